"""Fused LSTM cell on blocked weights — drop-in for ``brkernels.lstm`` plus the
north-star backward (BPTT) and weight-update passes.

Reference (``pkg/src/brkernels/lstm.py``, paper Alg. 2 / Eqs. 1-6): gates in
the order i, c, f, o (``lstm.py:28``); per time step every (ib_k, ib_n) item
is bias-initialised, accumulated with one BRGEMM over the C_b input blocks
and one over the K_b recurrent blocks, activated while hot and finished with
the state update (``lstm.py:268-317``); steps are separated by a barrier.

B200 mapping (all arithmetic in libbrk_sm100.so):

* the input projection of ALL steps is one grouped BRGEMM launch
  (``gx[t][n][g][k] = W_g x_t + b_g``, batch over C_b);
* every step is ONE fused launch (``brk_lstm_fwd_step``): the recurrent
  batch-reduce of all four gates lands in four TMEM accumulators side by side
  and the epilogue applies sigmoid/tanh and the cell update in registers;
* BPTT runs the mirrored fused step (``brk_lstm_bwd_step``) backwards in time,
  then dX, dW, dR and db are four grouped BRGEMM / column-sum launches over
  all T*N rows at once.

h, s, gates and gradients are stored in fp32 (as the reference); the tensor
cores take TF32 or BF16 inputs (``precision``), fp32 accumulation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import is_torch, require_cuda, stream_ptr
from ._grouped import addr_table, run_grouped
from .brgemm import get_default_precision
from .fc import default_minibatch_block
from .tensor import FP32, BlockedTensor, FetchCounter, LayoutError, block_weight_2d, clamp_block

GATE_NAMES = ("i", "c", "f", "o")


def sigmoid_block(buf):
    """In-place logistic sigmoid (host helper of the reference API, lstm.py:31-39)."""
    if is_torch(buf):
        return buf.sigmoid_()
    e = np.exp(-np.abs(buf))
    buf[...] = np.where(buf >= 0, 1.0 / (1.0 + e), e / (1.0 + e))
    return buf


def tanh_block(buf):
    """In-place tanh (host helper, lstm.py:42-45)."""
    if is_torch(buf):
        return buf.tanh_()
    np.tanh(buf, out=buf)
    return buf


@dataclass
class LstmCellWeights:
    """Dense weights: four (K, C) W_g, four (K, K) R_g, four (K,) biases (lstm.py:59-116)."""

    w_i: np.ndarray
    w_c: np.ndarray
    w_f: np.ndarray
    w_o: np.ndarray
    r_i: np.ndarray
    r_c: np.ndarray
    r_f: np.ndarray
    r_o: np.ndarray
    bias_i: np.ndarray
    bias_c: np.ndarray
    bias_f: np.ndarray
    bias_o: np.ndarray

    @property
    def hidden(self) -> int:
        return self.w_i.shape[0]

    @property
    def state(self) -> int:
        return self.w_i.shape[1]

    def validate(self) -> None:
        k, c = self.w_i.shape
        for g in GATE_NAMES:
            if getattr(self, f"w_{g}").shape != (k, c):
                raise LayoutError(f"w_{g} shape mismatch")
            if getattr(self, f"r_{g}").shape != (k, k):
                raise LayoutError(f"r_{g} shape mismatch")
            if getattr(self, f"bias_{g}").shape != (k,):
                raise LayoutError(f"bias_{g} shape mismatch")

    @classmethod
    def random(cls, rng: np.random.Generator, c: int, k: int, scale: float | None = None):
        """Uniform(-1, 1) * scale, scale 1/sqrt(C+K) by default (lstm.py:96-108 draw order)."""
        if scale is None:
            scale = 1.0 / np.sqrt(c + k)

        def m(rows, cols):
            return (rng.uniform(-1.0, 1.0, size=(rows, cols)) * scale).astype(FP32)

        def v(rows):
            return (rng.uniform(-1.0, 1.0, size=rows) * scale).astype(FP32)

        return cls(w_i=m(k, c), w_c=m(k, c), w_f=m(k, c), w_o=m(k, c),
                   r_i=m(k, k), r_c=m(k, k), r_f=m(k, k), r_o=m(k, k),
                   bias_i=v(k), bias_c=v(k), bias_f=v(k), bias_o=v(k))

    @classmethod
    def zeros(cls, c: int, k: int):
        return cls(**{f"w_{g}": np.zeros((k, c), FP32) for g in GATE_NAMES},
                   **{f"r_{g}": np.zeros((k, k), FP32) for g in GATE_NAMES},
                   **{f"bias_{g}": np.zeros(k, FP32) for g in GATE_NAMES})


@dataclass
class LstmParams:
    """Blocked descriptor: W_g [K_b][C_b][b_c][b_k], R_g [K_b][K_b][b_k][b_k] (lstm.py:119-198)."""

    w_i: BlockedTensor
    w_c: BlockedTensor
    w_f: BlockedTensor
    w_o: BlockedTensor
    r_i: BlockedTensor
    r_c: BlockedTensor
    r_f: BlockedTensor
    r_o: BlockedTensor
    bias_i: np.ndarray
    bias_c: np.ndarray
    bias_f: np.ndarray
    bias_o: np.ndarray
    t_steps: int
    n: int
    c: int
    k: int
    b_k: int
    b_c: int
    b_n: int

    @classmethod
    def from_dense(cls, weights: LstmCellWeights, t_steps: int, n: int, b_k: int | None = None,
                   b_c: int | None = None, b_n: int | None = None) -> "LstmParams":
        weights.validate()
        k, c = weights.w_i.shape
        b_k = clamp_block(k, 64 if b_k is None else b_k)
        b_c = clamp_block(c, 64 if b_c is None else b_c)
        b_n = default_minibatch_block(n) if b_n is None else b_n
        fields = {}
        for g in GATE_NAMES:
            fields[f"w_{g}"] = block_weight_2d(getattr(weights, f"w_{g}"), b_c, b_k)
            fields[f"r_{g}"] = block_weight_2d(getattr(weights, f"r_{g}"), b_k, b_k)
            fields[f"bias_{g}"] = getattr(weights, f"bias_{g}")
        params = cls(**fields, t_steps=t_steps, n=n, c=c, k=k, b_k=b_k, b_c=b_c, b_n=b_n)
        params.validate()
        return params

    def validate(self) -> None:
        for name, extent, block in (("K", self.k, self.b_k), ("C", self.c, self.b_c), ("N", self.n, self.b_n)):
            if block < 1 or extent % block:
                raise LayoutError(f"block {block} does not divide {name}={extent}")
        for g in GATE_NAMES:
            if getattr(self, f"w_{g}").logical_shape() != {"k": self.k, "c": self.c}:
                raise LayoutError(f"w_{g} blocked layout does not match dims")
            if getattr(self, f"r_{g}").logical_shape() != {"k": self.k, "c": self.k}:
                raise LayoutError(f"r_{g} blocked layout does not match dims")
            if tuple(getattr(self, f"bias_{g}").shape) != (self.k,):
                raise LayoutError(f"bias_{g} has wrong shape")

    @property
    def k_blocks(self) -> int:
        return self.k // self.b_k

    @property
    def c_blocks(self) -> int:
        return self.c // self.b_c

    @property
    def n_blocks(self) -> int:
        return self.n // self.b_n


@dataclass
class LstmStateSequence:
    """h[T][N][K], s[T][N][K] and (optionally) the activated gates per step."""

    h: object
    s: object
    gates: dict | None = None


@dataclass
class LstmGrads:
    """BPTT results: dx [T][N][C], dw/dr/db per gate (dense), dh0 / ds0 [N][K]."""

    dx: object
    dw: dict
    dr: dict
    db: dict
    dh0: object
    ds0: object


class _DeviceCell:
    """Device-resident fp32 copies of one LstmParams (cached on the params object,
    keyed on the source arrays' identity and content version, see _params_key)."""

    def __init__(self, params: LstmParams):
        torch = require_cuda()

        def dev(bt):
            return (bt.data if bt.on_device else torch.from_numpy(np.ascontiguousarray(bt.data))).to(
                "cuda", torch.float32)

        self.W = torch.stack([dev(getattr(params, f"w_{g}")) for g in GATE_NAMES]).contiguous()
        self.R = torch.stack([dev(getattr(params, f"r_{g}")) for g in GATE_NAMES]).contiguous()
        bias = [getattr(params, f"bias_{g}") for g in GATE_NAMES]
        self.bias = torch.cat([(b if is_torch(b) else torch.from_numpy(np.asarray(b, FP32))).float().reshape(-1)
                               for b in bias]).to("cuda").contiguous()


def _params_key(params: LstmParams) -> tuple:
    """Identity + content version of every source array of ``params``: device tensors
    by (storage pointer, autograd version counter, which in-place updates bump),
    host arrays by (address, crc32 of the bytes).  The device copies below are
    rebuilt whenever the key changes, so in-place weight updates (e.g. SGD on
    ``w_i.data`` or the bias arrays) are seen by the next call, as in the
    reference, which reads the params on every call."""
    import zlib

    key = []
    for g in GATE_NAMES:
        for a in (getattr(params, f"w_{g}").data, getattr(params, f"r_{g}").data, getattr(params, f"bias_{g}")):
            if is_torch(a):
                key.append((a.data_ptr(), a._version, tuple(a.shape), str(a.dtype)))
            else:
                arr = np.ascontiguousarray(a)
                key.append((arr.__array_interface__["data"][0], zlib.crc32(arr.view(np.uint8).reshape(-1)),
                            arr.shape, arr.dtype.str))
    return tuple(key)


def _device_cell(params: LstmParams) -> _DeviceCell:
    key = _params_key(params)
    cache = getattr(params, "_brk_device_cell", None)
    if cache is None or cache[0] != key:
        cache = (key, _DeviceCell(params))
        object.__setattr__(params, "_brk_device_cell", cache)
        object.__setattr__(params, "_brk_seq_cell", None)
    return cache[1]


def _to_dev(a, shape=None):
    torch = require_cuda()
    if a is None:
        return None
    t = a if is_torch(a) else torch.from_numpy(np.ascontiguousarray(np.asarray(a, FP32)))
    t = t.to("cuda", torch.float32).contiguous()
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise LayoutError(f"expected shape {shape}, got {tuple(t.shape)}")
    return t


class _SeqCell:
    """bf16 dense operands of the persistent sequence kernels (cached on the params):
    W_cat [4K][C] (rows g*K + k = W_g[k]), R_cat [4K][K], RT_cat [4K][K] (R_g^T), bias [4K]."""

    def __init__(self, params: LstmParams, dc: _DeviceCell):
        torch = require_cuda()
        k, c = params.k, params.c

        def dense(blk, cols):  # [K_b][X_b][b_x][b_k] -> (K, X)
            return blk.permute(0, 3, 1, 2).reshape(k, cols)

        w = [dense(dc.W[i], c) for i in range(4)]
        r = [dense(dc.R[i], k) for i in range(4)]
        self.w_cat = torch.cat(w).to(torch.bfloat16).contiguous()
        self.r_cat = torch.cat(r).to(torch.bfloat16).contiguous()
        self.rt_cat = torch.cat([ri.t() for ri in r]).to(torch.bfloat16).contiguous()
        self.bias = dc.bias


def _seq_cell(params: LstmParams) -> _SeqCell:
    dc = _device_cell(params)  # revalidates the source arrays (and drops a stale _SeqCell)
    cache = getattr(params, "_brk_seq_cell", None)
    if cache is None:
        cache = _SeqCell(params, dc)
        object.__setattr__(params, "_brk_seq_cell", cache)
    return cache


def _seq_ok(params: LstmParams, prec: str) -> bool:
    """The persistent sequence kernels (brk_lstm_seq_*) serve bf16 compute with
    N <= 256, K % 64 == 0, K <= 1024 and C % 64 == 0; other shapes and TF32 use
    the per-step kernels."""
    import os
    if os.environ.get("BRK_LSTM_SEQ", "1") == "0":
        return False
    return (prec == "bf16" and params.n <= 256 and params.k % 64 == 0 and params.k <= 1024
            and params.c % 64 == 0)


def _flags(k):
    torch = require_cuda()
    nbytes = _lib.load().brk_lstm_seq_flags_bytes(k)
    return torch.zeros(nbytes // 4, dtype=torch.int32, device="cuda")


def _forward_seq(params, xd, h0, s0, prec):
    from ._dense import gemm

    torch = require_cuda()
    T, N, C, K = params.t_steps, params.n, params.c, params.k
    sc = _seq_cell(params)
    xb = xd.to(torch.bfloat16)
    gx = torch.empty((T * N, 4 * K), dtype=torch.float32, device="cuda")
    gemm(xb, sc.w_cat, gx, bias=sc.bias)  # all steps' input projections: one BRGEMM launch
    h = torch.empty((T, N, K), dtype=torch.float32, device="cuda")
    s = torch.empty((T, N, K), dtype=torch.float32, device="cuda")
    gates = torch.empty((T, N, 4, K), dtype=torch.float32, device="cuda")
    h_bf = torch.empty((T + 1, N, K), dtype=torch.bfloat16, device="cuda")
    h_bf[0].copy_(h0)
    flags = _flags(K)
    rc = _lib.load().brk_lstm_seq_fwd(gx.data_ptr(), sc.r_cat.data_ptr(), s0.data_ptr() if s0 is not None else None,
                                      h_bf.data_ptr(), h.data_ptr(), s.data_ptr(), gates.data_ptr(), flags.data_ptr(),
                                      T, N, K, stream_ptr())
    _lib.check(rc, LayoutError)
    return h, s, gates, h_bf


def _compute(precision):
    prec = precision or get_default_precision()
    return prec, (_lib.BRK_COMPUTE_TF32 if prec == "tf32" else _lib.BRK_COMPUTE_BF16)


def _input_projection(dc: _DeviceCell, params: LstmParams, xd, prec):
    """gx[T*N][4][K] = x W_g^T + b_g for all steps: one grouped BRGEMM."""
    torch = require_cuda()
    T, N, C, K = params.t_steps, params.n, params.c, params.k
    b_c, b_k, cb, kb = params.b_c, params.b_k, params.c_blocks, params.k_blocks
    rows = T * N
    gx = torch.empty((rows, 4, K), dtype=torch.float32, device="cuda")
    # jobs (g, kb): C = gx[:, g, kb*b_k:+b_k] (rows x b_k, ldc = 4K); entries cb
    jg = torch.arange(4, device="cuda").repeat_interleave(kb)
    jk = torch.arange(kb, device="cuda").repeat(4)
    ci = torch.arange(cb, device="cuda")
    a_off = (((jg * kb + jk)[:, None] * cb) + ci[None, :]) * (b_c * b_k)
    b_off = (ci * b_c)[None, :].expand(4 * kb, cb)
    c_off = jg * K + jk * b_k
    run_grouped(a_ptrs=addr_table(dc.W, a_off.reshape(-1)), b_ptrs=addr_table(xd, b_off.reshape(-1).contiguous()),
                c_ptrs=addr_table(gx, c_off), m=b_k, n=rows, k=b_c, batch=cb,
                a_sk=b_k, a_sm=1, b_sn=C, b_sk=1, ldc=4 * K, in_bf16=False, out_bf16=False, precision=prec,
                bias=dc.bias, bias_offs=(jg * K + jk * b_k).contiguous(), exc=LayoutError)
    return gx


def lstm_forward(params: LstmParams, x, h_init=None, s_init=None, workers: int = 1, keep_gates: bool = False,
                 reduce_block: int | None = None, tile_force=None, fetch_counter: FetchCounter | None = None,
                 precision: str | None = None) -> LstmStateSequence:
    """Fused LSTM forward over x[T][N][C] (reference lstm.py:217-327)."""
    t_steps, n, c, k = params.t_steps, params.n, params.c, params.k
    if tuple(x.shape) != (t_steps, n, c):
        raise LayoutError(f"x has shape {tuple(x.shape)}, expected {(t_steps, n, c)}")
    if h_init is not None and tuple(h_init.shape) != (n, k) or s_init is not None and tuple(s_init.shape) != (n, k):
        raise LayoutError("h_init / s_init must have shape (N, K)")
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    params.validate()
    torch = require_cuda()
    host = not is_torch(x)
    prec, code = _compute(precision)
    dc = _device_cell(params)
    xd = _to_dev(x).reshape(t_steps * n, c)
    if _seq_ok(params, prec):
        h0 = _to_dev(h_init, (n, k)) if h_init is not None else torch.zeros((n, k), dtype=torch.float32,
                                                                             device="cuda")
        s0 = _to_dev(s_init, (n, k)) if s_init is not None else None
        h, s, gates, h_bf = _forward_seq(params, xd, h0, s0, prec)
        return _finish_forward(h, s, gates, host, keep_gates, h_bf)
    gx = _input_projection(dc, params, xd, prec).reshape(t_steps, n, 4, k)
    h = torch.empty((t_steps, n, k), dtype=torch.float32, device="cuda")
    s = torch.empty((t_steps, n, k), dtype=torch.float32, device="cuda")
    gates = torch.empty((t_steps, n, 4, k), dtype=torch.float32, device="cuda")
    h0 = _to_dev(h_init) if h_init is not None else torch.zeros((n, k), dtype=torch.float32, device="cuda")
    s0 = _to_dev(s_init) if s_init is not None else None
    lib = _lib.load()
    st = stream_ptr()
    for t in range(t_steps):
        hp = h[t - 1] if t > 0 else h0
        sp = s[t - 1] if t > 0 else s0
        rc = lib.brk_lstm_fwd_step(hp.data_ptr(), sp.data_ptr() if sp is not None else None, gx[t].data_ptr(),
                                   dc.R.data_ptr(), h[t].data_ptr(), s[t].data_ptr(), gates[t].data_ptr(),
                                   n, k, params.b_k, code, st)
        _lib.check(rc, LayoutError)
    return _finish_forward(h, s, gates, host, keep_gates, None)


def _finish_forward(h, s, gates, host, keep_gates, h_bf):
    if host:
        g_np = gates.cpu().numpy()
        gd = {g: np.ascontiguousarray(g_np[:, :, i]) for i, g in enumerate(GATE_NAMES)} if keep_gates else None
        seq = LstmStateSequence(h=h.cpu().numpy(), s=s.cpu().numpy(), gates=gd)
    else:
        gd = {g: gates[:, :, i] for i, g in enumerate(GATE_NAMES)} if keep_gates else None
        seq = LstmStateSequence(h=h, s=s, gates=gd)
    seq._brk_gates_dev = gates  # BPTT needs all four gates of every step
    seq._brk_h_bf = h_bf        # bf16 h_{t-1} of every step (sequence kernels): the dR operand
    return seq


def lstm_backward(params: LstmParams, x, seq: LstmStateSequence, dh, h_init=None, s_init=None,
                  precision: str | None = None, reducer=None) -> LstmGrads:
    """BPTT + weight update for the forward above (north star; oracle lstm_backward_reference).

    ``dh`` is dL/dh_t for every step [T][N][K].  Returns dense per-gate
    gradients dW_g (K, C), dR_g (K, K), db_g (K,), plus dx [T][N][C],
    dh0 / ds0 [N][K].  With a ``reducer`` (data parallel, dist.GradientReducer)
    each weight-gradient buffer's all-reduce is submitted as soon as its
    product is issued, overlapping the remaining BPTT products (dx, dh0).
    """
    t_steps, n, c, k = params.t_steps, params.n, params.c, params.k
    if tuple(dh.shape) != (t_steps, n, k):
        raise LayoutError(f"dh has shape {tuple(dh.shape)}, expected {(t_steps, n, k)}")
    torch = require_cuda()
    host = not is_torch(x)
    prec, code = _compute(precision)
    dc = _device_cell(params)
    gates = getattr(seq, "_brk_gates_dev", None)
    if gates is None:
        if seq.gates is None:
            raise LayoutError("lstm_backward needs the forward gates (run lstm_forward on the device)")
        gates = torch.stack([_to_dev(seq.gates[g]) for g in GATE_NAMES], dim=2).contiguous()
    hd = _to_dev(seq.h)
    sd = _to_dev(seq.s)
    dhd = _to_dev(dh)
    xd = _to_dev(x).reshape(t_steps * n, c)
    h0 = _to_dev(h_init) if h_init is not None else torch.zeros((n, k), dtype=torch.float32, device="cuda")
    s0 = _to_dev(s_init) if s_init is not None else None
    if _seq_ok(params, prec) and k % 32 == 0:
        out = _backward_seq(params, xd, hd, sd, gates, dhd, h0, s0, getattr(seq, "_brk_h_bf", None), reducer)
        if host:
            cpu = lambda t: t.cpu().numpy()  # noqa: E731
            out = LstmGrads(dx=cpu(out.dx), dw={g: cpu(v) for g, v in out.dw.items()},
                            dr={g: cpu(v) for g, v in out.dr.items()}, db={g: cpu(v) for g, v in out.db.items()},
                            dh0=cpu(out.dh0), ds0=cpu(out.ds0))
        return out
    dpre = torch.empty((t_steps, n, 4, k), dtype=torch.float32, device="cuda")
    ds = [torch.empty((n, k), dtype=torch.float32, device="cuda") for _ in range(2)]
    lib = _lib.load()
    st = stream_ptr()
    for t in range(t_steps - 1, -1, -1):
        nxt = dpre[t + 1].data_ptr() if t + 1 < t_steps else None
        ds_in = ds[(t + 1) % 2].data_ptr() if t + 1 < t_steps else None
        sp = sd[t - 1] if t > 0 else s0
        rc = lib.brk_lstm_bwd_step(nxt, dc.R.data_ptr(), dhd[t].data_ptr(), gates[t].data_ptr(), sd[t].data_ptr(),
                                   sp.data_ptr() if sp is not None else None, ds_in, dpre[t].data_ptr(),
                                   ds[t % 2].data_ptr(), n, k, params.b_k, code, st)
        _lib.check(rc, LayoutError)
    dh0 = torch.empty((n, k), dtype=torch.float32, device="cuda")
    _lib.check(lib.brk_lstm_recurrent_grad(dpre[0].data_ptr(), dc.R.data_ptr(), dh0.data_ptr(), n, k, params.b_k,
                                           code, st), LayoutError)
    ds0 = ds[0]
    rows = t_steps * n
    b_c, b_k, cb, kb = params.b_c, params.b_k, params.c_blocks, params.k_blocks
    dpre2 = dpre.reshape(rows, 4 * k)
    # dx[:, cb] = sum_(g,kb) dpre[:, g, kb] W_g[kb][cb]^T
    dx = torch.empty((rows, c), dtype=torch.float32, device="cuda")
    jc = torch.arange(cb, device="cuda")
    eg = torch.arange(4, device="cuda").repeat_interleave(kb)
    ek = torch.arange(kb, device="cuda").repeat(4)
    a_off = (((eg * kb + ek)[None, :] * cb) + jc[:, None]) * (b_c * b_k)
    b_off = (eg * k + ek * b_k)[None, :].expand(cb, 4 * kb)
    run_grouped(a_ptrs=addr_table(dc.W, a_off.reshape(-1)), b_ptrs=addr_table(dpre2, b_off.reshape(-1).contiguous()),
                c_ptrs=addr_table(dx, jc * b_c), m=b_c, n=rows, k=b_k, batch=4 * kb,
                a_sk=1, a_sm=b_k, b_sn=4 * k, b_sk=1, ldc=c, in_bf16=False, out_bf16=False, precision=prec,
                exc=LayoutError)
    # dW_g / dR_g: jobs (g, kb, cb) over one k = T*N reduction each (output in the blocked weight layout)
    h_prev = torch.cat([h0.reshape(1, n, k), hd[:-1]], dim=0).reshape(rows, k).contiguous()

    def weight_grad(src, cols, bcols):
        nblk = cols // bcols
        out = torch.empty((4, kb, nblk, bcols, b_k), dtype=torch.float32, device="cuda")
        jg2, jk2, jc2 = (t.reshape(-1) for t in torch.meshgrid(
            torch.arange(4, device="cuda"), torch.arange(kb, device="cuda"), torch.arange(nblk, device="cuda"),
            indexing="ij"))
        run_grouped(a_ptrs=addr_table(dpre2, jg2 * k + jk2 * b_k), b_ptrs=addr_table(src, jc2 * bcols),
                    c_ptrs=addr_table(out, ((jg2 * kb + jk2) * nblk + jc2) * (bcols * b_k)),
                    m=b_k, n=bcols, k=rows, batch=1, a_sk=4 * k, a_sm=1, b_sn=1, b_sk=cols, ldc=b_k,
                    in_bf16=False, out_bf16=False, precision=prec, exc=LayoutError)
        return out

    dw_blk = weight_grad(xd, c, b_c)
    dr_blk = weight_grad(h_prev, k, b_k)
    db = torch.empty(4 * k, dtype=torch.float32, device="cuda")
    _lib.check(lib.brk_colsum_blocked(dpre2.data_ptr(), None, None, db.data_ptr(), rows, 4 * k, rows, 4 * k,
                                      _lib.BRK_F32, st), LayoutError)
    if reducer is not None:
        reducer.submit([dw_blk, dr_blk, db])

    def dense(blk, cols):  # [4][K_b][X_b][b_x][b_k] -> 4 x (K, X)
        return [blk[i].permute(0, 3, 1, 2).reshape(k, cols) for i in range(4)]

    dws, drs = dense(dw_blk, c), dense(dr_blk, k)
    dbs = [db[i * k:(i + 1) * k] for i in range(4)]
    out = LstmGrads(dx=dx.reshape(t_steps, n, c), dw=dict(zip(GATE_NAMES, dws)), dr=dict(zip(GATE_NAMES, drs)),
                    db=dict(zip(GATE_NAMES, dbs)), dh0=dh0, ds0=ds0)
    if host:
        cpu = lambda t: t.cpu().numpy()  # noqa: E731
        out = LstmGrads(dx=cpu(out.dx), dw={g: cpu(v) for g, v in out.dw.items()},
                        dr={g: cpu(v) for g, v in out.dr.items()}, db={g: cpu(v) for g, v in out.db.items()},
                        dh0=cpu(dh0), ds0=cpu(ds0))
    return out


def _backward_seq(params, xd, hd, sd, gates, dhd, h0, s0, h_bf, reducer=None):
    """BPTT on the persistent backward kernel, then the step-independent
    products as single BRGEMM launches over all T*N rows: dx = dpre W,
    dW = dpre^T x, dR = dpre^T h_prev, dh0 = dpre_0 R, db = column sums."""
    from ._dense import gemm

    torch = require_cuda()
    T, N, C, K = params.t_steps, params.n, params.c, params.k
    sc = _seq_cell(params)
    lib = _lib.load()
    st = stream_ptr()
    dpre = torch.empty((T, N, 4, K), dtype=torch.bfloat16, device="cuda")
    ds0 = torch.empty((N, K), dtype=torch.float32, device="cuda")
    flags = _flags(K)
    rc = lib.brk_lstm_seq_bwd(dhd.data_ptr(), gates.data_ptr(), sd.data_ptr(),
                              s0.data_ptr() if s0 is not None else None, sc.rt_cat.data_ptr(), dpre.data_ptr(),
                              ds0.data_ptr(), flags.data_ptr(), T, N, K, st)
    _lib.check(rc, LayoutError)
    rows = T * N
    dp2 = dpre.reshape(rows, 4 * K)
    # weight gradients first: in data parallel their all-reduces overlap dx / dh0 below
    xb = xd.to(torch.bfloat16)
    if h_bf is None:
        h_bf = torch.empty((T + 1, N, K), dtype=torch.bfloat16, device="cuda")
        h_bf[0].copy_(h0)
        h_bf[1:].copy_(hd)
    hp = h_bf[:T].reshape(rows, K)
    dw = torch.empty((4 * K, C), dtype=torch.float32, device="cuda")
    gemm(dp2, xb, dw, a_t=True, b_t=True)                    # dW_cat = dpre^T x (reduction over T*N in TMEM)
    if reducer is not None:
        reducer.submit([dw])
    dr = torch.empty((4 * K, K), dtype=torch.float32, device="cuda")
    gemm(dp2, hp, dr, a_t=True, b_t=True)                    # dR_cat = dpre^T h_prev
    db = torch.empty(4 * K, dtype=torch.float32, device="cuda")
    _lib.check(lib.brk_colsum_blocked(dp2.data_ptr(), None, None, db.data_ptr(), rows, 4 * K, rows, 4 * K,
                                      _lib.BRK_BF16, st), LayoutError)
    if reducer is not None:
        reducer.submit([dr, db])
    dh0 = torch.empty((N, K), dtype=torch.float32, device="cuda")
    gemm(dp2[:N], sc.r_cat, dh0, b_t=True)                   # dh0 = dpre_0 [R_i; R_c; R_f; R_o]
    dx = torch.empty((rows, C), dtype=torch.float32, device="cuda")
    gemm(dp2, sc.w_cat, dx, b_t=True)                        # dx = dpre W_cat
    sl = lambda t: [t[i * K:(i + 1) * K] for i in range(4)]  # noqa: E731
    return LstmGrads(dx=dx.reshape(T, N, C), dw=dict(zip(GATE_NAMES, sl(dw))), dr=dict(zip(GATE_NAMES, sl(dr))),
                     db=dict(zip(GATE_NAMES, sl(db))), dh0=dh0, ds0=ds0)
