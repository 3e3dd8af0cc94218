"""Fully-connected layer on blocked layouts — drop-in for ``brkernels.fc`` plus the
north-star backward-data, weight-update and bias passes.

Reference behaviour (``pkg/src/brkernels/fc.py``):

* ``fc_forward`` (fc.py:99-163): ``Y[ib_n][ib_k] = g(sum_cb W[ib_k][cb] X[ib_n][cb])``
  — one BRGEMM per output block with batch C_b, activation applied on the hot
  block.  Here every output block of the pass is one tile of ONE launch; the
  activation (and the new optional bias) is fused into the TMEM epilogue.
* The reference has no bias, no backward and no weight update; those follow
  the CPU restatement in ``oracle/``:
  ``dX = W^T dZ``, ``dW = dZ X^T``, ``db = sum_n dZ`` with ``dZ = dY * g'(Z)``.

Two native paths (no CPU fallback):

* engine (TMA -> tcgen05, persistent, warp-specialised) for bf16 storage with
  b_n = b_c = b_k = 64 and N, C, K multiples of 128 — the benchmark layout;
* grouped batch-list BRGEMM (``brk_brgemm_grouped``) for every other blocking
  and for fp32 storage (TF32 or BF16 tensor-core inputs).
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from enum import Enum

import numpy as np

from . import _lib
from ._device import is_torch, require_cuda, stream_ptr
from ._grouped import addr_table, run_grouped
from .brgemm import get_default_precision
from .tensor import FP32, BlockedTensor, FetchCounter, LayoutError, block_weight_2d, clamp_block


def _sigmoid_host(buf: np.ndarray) -> np.ndarray:
    e = np.exp(-np.abs(buf))
    buf[...] = np.where(buf >= 0, 1.0 / (1.0 + e), e / (1.0 + e))
    return buf


class Activation(Enum):
    """Fused output activation (reference fc.py:29-40)."""

    IDENTITY = "identity"
    RELU = "relu"
    SIGMOID = "sigmoid"

    @property
    def code(self) -> int:
        return {"identity": 0, "relu": 1, "sigmoid": 2}[self.value]

    def apply(self, buf):
        """In-place activation on a block (host helper kept for API compatibility)."""
        if is_torch(buf):
            if self is Activation.RELU:
                buf.clamp_(min=0)
            elif self is Activation.SIGMOID:
                buf.sigmoid_()
            return buf
        if self is Activation.RELU:
            np.maximum(buf, 0.0, out=buf)
        elif self is Activation.SIGMOID:
            _sigmoid_host(buf)
        return buf


def default_minibatch_block(extent: int, cap: int = 64) -> int:
    """Largest divisor of ``extent`` not above ``cap`` (reference lstm.py:51-56)."""
    b = min(extent, cap)
    while extent % b:
        b -= 1
    return b


@dataclass
class FcParams:
    """Blocked (K, C) weights, dims, blocking, activation and optional bias (fc.py:43-96)."""

    w: BlockedTensor
    n: int
    c: int
    k: int
    b_n: int
    b_c: int
    b_k: int
    activation: Activation = Activation.IDENTITY
    bias: object = None  # (K,) fp32, host or device; north-star extension

    @classmethod
    def from_dense(cls, w_dense, n: int, b_n: int | None = None, b_c: int | None = None,
                   b_k: int | None = None, activation: Activation = Activation.IDENTITY,
                   bias=None) -> "FcParams":
        k, c = w_dense.shape
        b_k = clamp_block(k, 64 if b_k is None else b_k)
        b_c = clamp_block(c, 64 if b_c is None else b_c)
        b_n = default_minibatch_block(n) if b_n is None else b_n
        params = cls(w=block_weight_2d(w_dense, b_c, b_k), n=n, c=c, k=k, b_n=b_n, b_c=b_c,
                     b_k=b_k, activation=activation, bias=bias)
        params.validate()
        return params

    def validate(self) -> None:
        for name, extent, block in (("N", self.n, self.b_n), ("C", self.c, self.b_c), ("K", self.k, self.b_k)):
            if block < 1 or extent % block:
                raise LayoutError(f"block {block} does not divide {name}={extent}")
        if self.w.logical_shape() != {"k": self.k, "c": self.c}:
            raise LayoutError("blocked weights do not match (K, C) dims")
        if self.bias is not None and tuple(self.bias.shape) != (self.k,):
            raise LayoutError(f"bias must have shape ({self.k},), got {tuple(self.bias.shape)}")

    @property
    def k_blocks(self) -> int:
        return self.k // self.b_k

    @property
    def c_blocks(self) -> int:
        return self.c // self.b_c

    @property
    def n_blocks(self) -> int:
        return self.n // self.b_n

    def to(self, device: str = "cuda", dtype=None) -> "FcParams":
        """Device copy of the weights (``dtype`` e.g. torch.bfloat16); bias stays fp32."""
        torch = require_cuda()
        bias = self.bias
        if bias is not None:
            bias = (bias if is_torch(bias) else torch.from_numpy(np.asarray(bias, FP32))).to(device).float()
        return replace(self, w=self.w.to(device, dtype), bias=bias)


# ---------------------------------------------------------------------------
# device staging
# ---------------------------------------------------------------------------
def _storage_dtype(precision: str):
    torch = require_cuda()
    return torch.bfloat16 if precision == "bf16" else torch.float32


def _resolve(precision, *tensors):
    """Pick the compute precision: device bf16 data forces bf16; else the default."""
    torch = require_cuda()
    for t in tensors:
        if t is not None and t.on_device and t.data.dtype == torch.bfloat16:
            return "bf16"
    return precision or get_default_precision()


def _stage(bt: BlockedTensor, dtype):
    """Device tensor of a blocked tensor in the compute storage dtype (no copy if already there)."""
    if bt.on_device and bt.data.dtype == dtype:
        return bt.data.contiguous()
    return bt.to("cuda", dtype).data


def _stage_bias(bias):
    torch = require_cuda()
    if bias is None:
        return None
    t = bias if is_torch(bias) else torch.from_numpy(np.ascontiguousarray(bias, dtype=FP32))
    return t.to("cuda", torch.float32).contiguous()


def _engine_ok(p: FcParams, dtype) -> bool:
    """The TMA / tcgen05 engine serves 64-element blocks with N, C, K multiples of 128:
    bf16 storage on kind::f16, fp32 storage on kind::tf32 (other blockings take the
    grouped BRGEMM path, which follows the reference's batch lists directly)."""
    torch = require_cuda()
    return (dtype in (torch.bfloat16, torch.float32) and p.b_n == 64 and p.b_c == 64 and p.b_k == 64
            and p.n % 128 == 0 and p.c % 128 == 0 and p.k % 128 == 0)


def _dcode(dt) -> int:
    torch = require_cuda()
    return _lib.BRK_BF16 if dt == torch.bfloat16 else _lib.BRK_F32


def tf32_operand(t):
    """fp32 operand of a TF32 engine pass, rounded to TF32 (round-to-nearest, cvt.rna) into
    a new device tensor (``brk_round_tf32``): the tensor cores read fp32 bit patterns
    truncated to TF32, whose bias (~7e-4 of a dot product) would eat most of the 1e-3
    TF32 tolerance; rounded inputs give ~3e-4.  bf16 tensors pass through."""
    torch = require_cuda()
    if t is None or t.dtype != torch.float32:
        return t
    out = torch.empty_like(t)
    _lib.check(_lib.load().brk_round_tf32(t.data_ptr(), out.data_ptr(), t.numel(), stream_ptr()), LayoutError)
    return out


def _act_blocked(data) -> BlockedTensor:
    return BlockedTensor(data, n_outer=2, logical_dims={"n": (0, 2), "c": (1, 3)})


def _workers_ok(workers):
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")


# ---------------------------------------------------------------------------
# passes
# ---------------------------------------------------------------------------
def fc_forward(params: FcParams, x: BlockedTensor, workers: int = 1, reduce_block: int | None = None,
               tile_force: tuple[int, int] | None = None, fetch_counter: FetchCounter | None = None,
               precision: str | None = None) -> BlockedTensor:
    """Y = g(W X + b) over X[N_b][C_b][b_n][b_c]; returns Y[N_b][K_b][b_n][b_k].

    ``workers`` / ``reduce_block`` / ``tile_force`` / ``fetch_counter`` are the
    reference's CPU scheduling knobs: validated and otherwise ignored (the
    whole C_b reduction of a tile stays in TMEM, so chunking never applies).
    """
    params.validate()
    if x.logical_shape() != {"n": params.n, "c": params.c}:
        raise LayoutError(f"input layout {x.logical_shape()} does not match N={params.n}, C={params.c}")
    if x.inner_shape != (params.b_n, params.b_c):
        raise LayoutError(f"input blocking {x.inner_shape} does not match ({params.b_n}, {params.b_c})")
    _workers_ok(workers)
    torch = require_cuda()
    host = not x.on_device
    prec = _resolve(precision, x, params.w)
    dt = _storage_dtype(prec)
    xd, wd = _stage(x, dt), _stage(params.w, dt)
    bias = _stage_bias(params.bias)
    nb, kb, cb = params.n_blocks, params.k_blocks, params.c_blocks
    y = torch.empty((nb, kb, params.b_n, params.b_k), dtype=dt, device="cuda")
    if _engine_ok(params, dt):
        xd, wd = tf32_operand(xd), tf32_operand(wd)
        rc = _lib.load().brk_fc_fwd(xd.data_ptr(), wd.data_ptr(), bias.data_ptr() if bias is not None else None,
                                    y.data_ptr(), params.n, params.c, params.k, 64, 64, 64,
                                    params.activation.code, _dcode(dt), stream_ptr())
        _lib.check(rc, LayoutError)
    else:
        b_n, b_c, b_k = params.b_n, params.b_c, params.b_k
        dev = "cuda"
        jn = torch.arange(nb, device=dev).repeat_interleave(kb)      # job -> ib_n
        jk = torch.arange(kb, device=dev).repeat(nb)                 # job -> ib_k
        ci = torch.arange(cb, device=dev)
        a_off = (jk[:, None] * cb + ci[None, :]) * (b_c * b_k)
        b_off = (jn[:, None] * cb + ci[None, :]) * (b_n * b_c)
        c_off = (jn * kb + jk) * (b_n * b_k)
        run_grouped(a_ptrs=addr_table(wd, a_off.reshape(-1)), b_ptrs=addr_table(xd, b_off.reshape(-1)),
                    c_ptrs=addr_table(y, c_off), m=b_k, n=b_n, k=b_c, batch=cb,
                    a_sk=b_k, a_sm=1, b_sn=b_c, b_sk=1, ldc=b_k,
                    in_bf16=dt == torch.bfloat16, out_bf16=dt == torch.bfloat16, precision=prec,
                    bias=bias, bias_offs=(jk * b_k).contiguous() if bias is not None else None,
                    act=params.activation.code, exc=LayoutError)
    out = BlockedTensor(y, n_outer=2, logical_dims={"n": (0, 2), "k": (1, 3)})
    return out.to("cpu") if host else out


def fc_backward_data(params: FcParams, dz: BlockedTensor, mask: BlockedTensor | None = None,
                     precision: str | None = None) -> BlockedTensor:
    """dX = (W^T dZ) * (mask > 0): dZ[N_b][K_b][b_n][b_k] -> dX[N_b][C_b][b_n][b_c].

    ``mask`` (optional) is the previous layer's activation output in the dX
    layout; passing it fuses that layer's ReLU derivative into this epilogue.
    """
    params.validate()
    if dz.logical_shape() != {"n": params.n, "k": params.k} or dz.inner_shape != (params.b_n, params.b_k):
        raise LayoutError(f"dz layout {dz.logical_shape()}/{dz.inner_shape} does not match the layer")
    if mask is not None and (mask.logical_shape() != {"n": params.n, "c": params.c}
                             or mask.inner_shape != (params.b_n, params.b_c)):
        raise LayoutError("mask layout does not match the layer input")
    torch = require_cuda()
    host = not dz.on_device
    prec = _resolve(precision, dz, params.w)
    dt = _storage_dtype(prec)
    dzd, wd = _stage(dz, dt), _stage(params.w, dt)
    md = _stage(mask, dt) if mask is not None else None
    nb, kb, cb = params.n_blocks, params.k_blocks, params.c_blocks
    dx = torch.empty((nb, cb, params.b_n, params.b_c), dtype=dt, device="cuda")
    if _engine_ok(params, dt):
        dzd, wd = tf32_operand(dzd), tf32_operand(wd)
        rc = _lib.load().brk_fc_bwd_data(dzd.data_ptr(), wd.data_ptr(), md.data_ptr() if md is not None else None,
                                         dx.data_ptr(), None, params.n, params.c, params.k, 64, 64, 64,
                                         _dcode(dt), stream_ptr())
        _lib.check(rc, LayoutError)
    else:
        b_n, b_c, b_k = params.b_n, params.b_c, params.b_k
        dev = "cuda"
        jn = torch.arange(nb, device=dev).repeat_interleave(cb)
        jc = torch.arange(cb, device=dev).repeat(nb)
        ki = torch.arange(kb, device=dev)
        a_off = (ki[None, :] * cb + jc[:, None]) * (b_c * b_k)       # W[kb][cb] viewed (b_k x b_c)
        b_off = (jn[:, None] * kb + ki[None, :]) * (b_n * b_k)       # dZ[nb][kb]
        c_off = (jn * cb + jc) * (b_n * b_c)
        run_grouped(a_ptrs=addr_table(wd, a_off.reshape(-1)), b_ptrs=addr_table(dzd, b_off.reshape(-1)),
                    c_ptrs=addr_table(dx, c_off), m=b_c, n=b_n, k=b_k, batch=kb,
                    a_sk=1, a_sm=b_k, b_sn=b_k, b_sk=1, ldc=b_c,
                    in_bf16=dt == torch.bfloat16, out_bf16=dt == torch.bfloat16, precision=prec,
                    mask_ptrs=addr_table(md, c_off) if md is not None else None, exc=LayoutError)
    out = _act_blocked(dx)
    return out.to("cpu") if host else out


def fc_weight_update(params: FcParams, x: BlockedTensor, dz: BlockedTensor, lr: float | None = None,
                     precision: str | None = None) -> BlockedTensor:
    """dW = dZ X^T in the weight layout [K_b][C_b][b_c][b_k] (fp32).

    With ``lr`` the SGD step ``W -= lr * dW`` is applied to ``params.w`` in
    place (fused into the epilogue on the engine path) — device weights only.
    """
    params.validate()
    if x.logical_shape() != {"n": params.n, "c": params.c} or x.inner_shape != (params.b_n, params.b_c):
        raise LayoutError("input layout does not match the layer")
    if dz.logical_shape() != {"n": params.n, "k": params.k} or dz.inner_shape != (params.b_n, params.b_k):
        raise LayoutError("dz layout does not match the layer")
    torch = require_cuda()
    host = not x.on_device
    prec = _resolve(precision, x, dz, params.w)
    dt = _storage_dtype(prec)
    xd, dzd = _stage(x, dt), _stage(dz, dt)
    nb, kb, cb = params.n_blocks, params.k_blocks, params.c_blocks
    dw = torch.empty((kb, cb, params.b_c, params.b_k), dtype=torch.float32, device="cuda")
    sgd_w = None
    if lr is not None:
        if not params.w.on_device:
            raise LayoutError("the fused SGD update needs device-resident weights (FcParams.to)")
        sgd_w = params.w.data
    if _engine_ok(params, dt):
        lib = _lib.load()
        ws = upd_workspace(params.n, params.c, params.k)
        fused = sgd_w is not None and sgd_w.dtype == torch.bfloat16 and dt == torch.bfloat16
        xd, dzd = tf32_operand(xd), tf32_operand(dzd)
        rc = lib.brk_fc_upd(xd.data_ptr(), dzd.data_ptr(), dw.data_ptr(),
                            sgd_w.data_ptr() if fused else None, float(lr or 0.0) if fused else 0.0,
                            None, 0, None, None, 0.0, ws.data_ptr(), ws.numel(),
                            params.n, params.c, params.k, 64, 64, 64, _dcode(dt), stream_ptr())
        _lib.check(rc, LayoutError)
        if sgd_w is not None and not fused:
            rc = lib.brk_sgd_apply(sgd_w.data_ptr(), dw.data_ptr(), float(lr), dw.numel(),
                                   _dcode(sgd_w.dtype), stream_ptr())
            _lib.check(rc, LayoutError)
    else:
        b_n, b_c, b_k = params.b_n, params.b_c, params.b_k
        dev = "cuda"
        jk = torch.arange(kb, device=dev).repeat_interleave(cb)
        jc = torch.arange(cb, device=dev).repeat(kb)
        ni = torch.arange(nb, device=dev)
        a_off = (ni[None, :] * kb + jk[:, None]) * (b_n * b_k)      # dZ[nb][kb] as (k=b_n, m=b_k)
        b_off = (ni[None, :] * cb + jc[:, None]) * (b_n * b_c)      # X[nb][cb]^T as (n=b_c, k=b_n)
        c_off = (jk * cb + jc) * (b_c * b_k)
        run_grouped(a_ptrs=addr_table(dzd, a_off.reshape(-1)), b_ptrs=addr_table(xd, b_off.reshape(-1)),
                    c_ptrs=addr_table(dw, c_off), m=b_k, n=b_c, k=b_n, batch=nb,
                    a_sk=b_k, a_sm=1, b_sn=1, b_sk=b_c, ldc=b_k,
                    in_bf16=dt == torch.bfloat16, out_bf16=False, precision=prec, exc=LayoutError)
        if sgd_w is not None:
            rc = _lib.load().brk_sgd_apply(sgd_w.data_ptr(), dw.data_ptr(), float(lr), dw.numel(),
                                           _lib.BRK_BF16 if sgd_w.dtype == torch.bfloat16 else _lib.BRK_F32,
                                           stream_ptr())
            _lib.check(rc, LayoutError)
    out = BlockedTensor(dw, n_outer=2, logical_dims={"k": (0, 3), "c": (1, 2)})
    return out.to("cpu") if host else out


_BIAS_WS: dict = {}
_UPD_WS: dict = {}


def upd_workspace(n: int, c: int, k: int):
    """Cached, zero-initialised split-K workspace of the weight-update engine pass."""
    torch = require_cuda()
    key = (torch.cuda.current_device(), n, c, k)
    ws = _UPD_WS.get(key)
    if ws is None:
        nbytes = max(int(_lib.load().brk_fc_upd_workspace(n, c, k)), 16)
        ws = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        _UPD_WS[key] = ws
    return ws


def fc_bias_grad(dy: BlockedTensor, y: BlockedTensor | None = None):
    """db = sum_n dZ with dZ = dY * (Y > 0) when ``y`` is given (ReLU layers).

    Returns ``(db, dz)``; ``dz`` is ``dy`` itself when no mask applies.
    Deterministic (fixed summation order).
    """
    names = dy.logical_dims
    if len(names) != 2 or "n" not in names or dy.n_outer != 2 or len(dy.shape) != 4:
        raise LayoutError("dy must be an [N_b][K_b][b_n][b_k] blocked tensor")
    if y is not None and (y.shape != dy.shape):
        raise LayoutError("y must match dy's layout")
    torch = require_cuda()
    host = not dy.on_device
    dt = dy.data.dtype if dy.on_device else torch.float32
    dyd = _stage(dy, dt)
    yd = _stage(y, dt) if y is not None else None
    n_b, k_b, b_n, b_k = dyd.shape
    N, K = n_b * b_n, k_b * b_k
    db = torch.empty(K, dtype=torch.float32, device="cuda")
    dz = torch.empty_like(dyd) if yd is not None else dyd
    lib = _lib.load()
    if dt == torch.bfloat16 and b_n == 64 and b_k == 64 and N % 16 == 0:
        key = (torch.cuda.current_device(), K)
        ws = _BIAS_WS.get(key)
        if ws is None:
            ws = torch.zeros(lib.brk_fc_bias_grad_workspace(K), dtype=torch.uint8, device="cuda")
            _BIAS_WS[key] = ws
        rc = lib.brk_fc_bias_grad(dyd.data_ptr(), yd.data_ptr() if yd is not None else None,
                                  dz.data_ptr() if yd is not None else None, db.data_ptr(), ws.data_ptr(),
                                  N, K, 64, 64, None, 0.0, stream_ptr())
    else:
        rc = lib.brk_colsum_blocked(dyd.data_ptr(), yd.data_ptr() if yd is not None else None,
                                    dz.data_ptr() if yd is not None else None, db.data_ptr(), N, K, b_n, b_k,
                                    _lib.BRK_BF16 if dt == torch.bfloat16 else _lib.BRK_F32, stream_ptr())
    _lib.check(rc, LayoutError)
    # dz is the gradient of a layer OUTPUT: label its feature dim "k" (the
    # layout bwd-data / weight-update expect), whatever dy was called
    dz_bt = BlockedTensor(dz, n_outer=2, logical_dims={"n": (0, 2), "k": (1, 3)})
    if host:
        return db.cpu().numpy(), dz_bt.to("cpu")
    return db, dz_bt
