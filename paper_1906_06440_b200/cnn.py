"""Direct convolution on blocked layouts — drop-in for ``brkernels.cnn`` plus the
north-star backward-data and weight-update passes.

Reference algorithm (``pkg/src/brkernels/cnn.py:201-334``, paper Alg. 4): for
every (image, output-channel block, output row, pixel tile) the weight and
input sub-blocks of all (r, s, c) triples form ONE batch-reduce GEMM, so the
output tile is accumulated without ever being reloaded.  Here every such
output block of a pass is one job of ONE grouped tcgen05 BRGEMM launch
(``brk_brgemm_grouped``) whose device-side batch lists are exactly the
reference's pointer lists (``cnn.py:241-252, 304-310``):

* fwd   job (img, kb, oj): C = O[img][kb][oj][:]            (Q x b_k)
        entries (c_b, r, s): A = W[kb][c_b][r][s]            (b_c x b_k)
                              B = I_pad[img][c_b][oj*str+r][s::str]  (Q x b_c, row stride str*b_c)
* bwd   "dual convolution": dI = conv(dO dilated by the stride
        and padded by R-1-pad, flipped W with C<->K swapped); unpadded 1x1
        stride-s layers scatter a 1x1 GEMM to the strided input positions.
* upd   job (kb, c_b, r, s): C = dW[kb][c_b][r][s]           (b_c x b_k)
        entries (img, oj):   A = dO[img][kb][oj]             (Q x b_k)
                             B = I_pad[img][c_b][oj*str+r][s::str]^T (b_c x Q)

Zero padding is materialised on the device (the reference pads by copy,
``cnn.py:234-237``).  All arithmetic runs in libbrk_sm100.so; there is no CPU
fallback.  Strategies / worker counts of the CPU reference only reorder work
and are accepted for API compatibility.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

import os

from . import _lib
from ._device import require_cuda, stream_ptr
from ._grouped import addr_table, run_grouped
from .brgemm import get_default_precision
from .tensor import (
    BlockedTensor,
    LayoutError,
    clamp_block,
    make_conv_output,
)

WEIGHT_SLICE_BUDGET = 512 * 1024
STRATEGY_WEIGHT_BUDGET = 1024 * 1024
DEFAULT_CHANNEL_BLOCK = 64


class StrategyKind(Enum):
    MINIBATCH_FIRST = "minibatch"
    TASK_GRID = "task-grid"
    FEATURE_MAP_FIRST = "feature-map"


@dataclass(frozen=True)
class ParallelStrategy:
    kind: StrategyKind
    workers: int = 1


@dataclass
class ConvSpec:
    """Convolution descriptor plus blocking (reference cnn.py:52-135).

    Same-padding ((r-1)/2) by default for odd filters; channel blocks default
    to min(64, extent); ``b_q`` / ``cb_chunk`` are the CPU tiling knobs
    (validated; the GPU reduces all of C_b, R, S in one TMEM chain).
    """

    n: int
    c: int
    k: int
    h: int
    w: int
    r: int
    s: int
    stride: int = 1
    pad_h: int | None = None
    pad_w: int | None = None
    b_c: int | None = None
    b_k: int | None = None
    b_q: int | None = None
    cb_chunk: int | None = None

    def __post_init__(self):
        if self.pad_h is None:
            if self.r % 2 == 0:
                raise LayoutError(f"even filter height r={self.r} needs an explicit pad_h")
            self.pad_h = (self.r - 1) // 2
        if self.pad_w is None:
            if self.s % 2 == 0:
                raise LayoutError(f"even filter width s={self.s} needs an explicit pad_w")
            self.pad_w = (self.s - 1) // 2
        self.b_c = clamp_block(self.c, DEFAULT_CHANNEL_BLOCK if self.b_c is None else self.b_c)
        self.b_k = clamp_block(self.k, DEFAULT_CHANNEL_BLOCK if self.b_k is None else self.b_k)
        self.validate()

    def validate(self) -> None:
        for name in ("n", "c", "k", "h", "w", "r", "s"):
            if getattr(self, name) < 1:
                raise LayoutError(f"{name} must be >= 1, got {getattr(self, name)}")
        if self.stride < 1:
            raise LayoutError(f"stride must be >= 1, got {self.stride}")
        if self.pad_h < 0 or self.pad_w < 0:
            raise LayoutError("padding must be >= 0")
        if self.c % self.b_c:
            raise LayoutError(f"b_c={self.b_c} does not divide C={self.c}")
        if self.k % self.b_k:
            raise LayoutError(f"b_k={self.b_k} does not divide K={self.k}")
        if self.h + 2 * self.pad_h < self.r or self.w + 2 * self.pad_w < self.s:
            raise LayoutError("filter larger than padded input")
        if self.out_h < 1 or self.out_w < 1:
            raise LayoutError("output spatial extents must be >= 1")
        if self.b_q is not None and self.b_q < 1:
            raise LayoutError(f"b_q must be >= 1, got {self.b_q}")
        if self.cb_chunk is not None and (self.cb_chunk < 1 or self.c_blocks % self.cb_chunk):
            raise LayoutError(f"cb_chunk={self.cb_chunk} must divide C_b={self.c_blocks}")

    @property
    def out_h(self) -> int:
        return (self.h + 2 * self.pad_h - self.r) // self.stride + 1

    @property
    def out_w(self) -> int:
        return (self.w + 2 * self.pad_w - self.s) // self.stride + 1

    @property
    def c_blocks(self) -> int:
        return self.c // self.b_c

    @property
    def k_blocks(self) -> int:
        return self.k // self.b_k

    @property
    def weight_bytes(self) -> int:
        return self.k * self.c * self.r * self.s * 4


@dataclass(frozen=True)
class PixelCollapse:
    applied: bool
    extent: int


def collapse_pixels(spec: ConvSpec) -> PixelCollapse:
    """1x1 unit-stride unpadded convolutions walk P*Q pixels as one extent (cnn.py:146-155)."""
    ok = spec.r == 1 and spec.s == 1 and spec.stride == 1 and spec.pad_h == 0 and spec.pad_w == 0
    return PixelCollapse(applied=ok, extent=spec.out_h * spec.out_w if ok else spec.out_w)


def choose_strategy(spec: ConvSpec, workers: int, cache_budget: int = STRATEGY_WEIGHT_BUDGET) -> ParallelStrategy:
    """Task-assignment strategy of the CPU reference (cnn.py:158-176); never changes results."""
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if spec.n >= workers:
        kind = StrategyKind.MINIBATCH_FIRST
    elif spec.weight_bytes > cache_budget:
        kind = StrategyKind.FEATURE_MAP_FIRST
    else:
        kind = StrategyKind.TASK_GRID
    return ParallelStrategy(kind=kind, workers=workers)


def _check_layouts(spec: ConvSpec, inp: BlockedTensor, wgt: BlockedTensor) -> None:
    want_in = {"n": spec.n, "c": spec.c, "h": spec.h, "w": spec.w}
    if inp.logical_shape() != want_in or inp.inner_shape != (spec.b_c,):
        raise LayoutError(f"input layout {inp.logical_shape()}/{inp.inner_shape} does not match spec")
    want_w = {"k": spec.k, "c": spec.c, "r": spec.r, "s": spec.s}
    if wgt.logical_shape() != want_w or wgt.inner_shape != (spec.b_c, spec.b_k):
        raise LayoutError(f"weight layout {wgt.logical_shape()}/{wgt.inner_shape} does not match spec")


def _dtype(precision, *tensors):
    torch = require_cuda()
    for t in tensors:
        if t is not None and t.on_device and t.data.dtype == torch.bfloat16:
            return "bf16", torch.bfloat16
    prec = precision or get_default_precision()
    return prec, (torch.bfloat16 if prec == "bf16" else torch.float32)


def _stage(bt: BlockedTensor, dt):
    if bt.on_device and bt.data.dtype == dt:
        return bt.data.contiguous()
    return bt.to("cuda", dt).data


def _pad_device(x, pad_h, pad_w):
    """[N][C_b][H][W][b_c] -> zero-padded copy (device plumbing)."""
    torch = require_cuda()
    if not pad_h and not pad_w:
        return x
    n, cb, h, w, bc = x.shape
    out = torch.zeros((n, cb, h + 2 * pad_h, w + 2 * pad_w, bc), dtype=x.dtype, device=x.device)
    out[:, :, pad_h:pad_h + h, pad_w:pad_w + w] = x
    return out


def _engine_ok(spec: "ConvSpec", dt, pass_: str, engine: bool | None) -> bool:
    """Whether a pass runs on the implicit-GEMM tcgen05 engine (brk_conv_*):
    bf16 or fp32 (TF32) storage, 64-channel blocks, stride 1 or 1x1 stride 2 (include/brk.h).
    Everything else (other blockings, the 3-channel stem) runs on the grouped BRGEMM path,
    which follows the reference's batch lists directly."""
    torch = require_cuda()
    if engine is False or os.environ.get("BRK_CONV_ENGINE", "1") == "0":
        return False
    dt_ok = dt in (torch.bfloat16, torch.float32)
    ok = (dt_ok and spec.b_c == 64 and spec.b_k == 64 and spec.c % 64 == 0
          and spec.k % 64 == 0 and max(spec.pad_h, spec.pad_w) <= 15 and max(spec.r, spec.s) <= 16)
    if ok and spec.stride == 1:
        if pass_ == "bwd":
            ok = spec.out_h == spec.h and spec.out_w == spec.w
    elif ok:
        ok = spec.stride == 2 and spec.r == 1 and spec.s == 1 and spec.pad_h == 0 and spec.pad_w == 0
        if ok and pass_ == "bwd":
            ok = spec.h == 2 * spec.out_h and spec.w == 2 * spec.out_w
    if engine and not ok:
        raise LayoutError(f"conv {pass_}: shape/dtype not served by the engine path")
    return ok


def _small_ok(spec: "ConvSpec", dt, engine: bool | None) -> bool:
    """Small-channel convs (the 3-channel ResNet stem): explicit im2col + the dense
    tcgen05 GEMM (brk_conv_im2col / brk_gemm_dense / brk_conv_col2im) instead of a
    64-channel im2col box that would be almost all padding.  bf16, K = 64."""
    torch = require_cuda()
    if engine is False or os.environ.get("BRK_CONV_ENGINE", "1") == "0":
        return False
    return dt == torch.bfloat16 and spec.c < 64 and spec.k == 64 and spec.b_k == 64


def _s2d_ok(spec: "ConvSpec", dt, engine: bool | None) -> bool:
    """Stride-2 convs over <= 4 channels in one block (the ResNet-50 stem): space-to-depth
    unfold to 64 channels + the implicit-GEMM engine (brk_conv_s2d_*, csrc/brk_conv_s2d.cu).
    BRK_CONV_S2D=0 selects the explicit-im2col path instead (A/B diagnostics)."""
    torch = require_cuda()
    if engine is False or os.environ.get("BRK_CONV_ENGINE", "1") == "0" or os.environ.get("BRK_CONV_S2D", "1") == "0":
        return False
    if not (dt == torch.bfloat16 and spec.stride == 2 and spec.c <= 4 and spec.b_c == spec.c and spec.b_k == 64
            and spec.k % 64 == 0):
        return False
    return _lib.load().brk_conv_s2d_shape(*_s2d_args(spec), None) == 0


def _s2d_args(spec: "ConvSpec"):
    return (spec.n, spec.c, spec.k, spec.h, spec.w, spec.r, spec.s, spec.pad_h, spec.pad_w)


def _s2d_workspace(spec: "ConvSpec"):
    return _workspace(int(_lib.load().brk_conv_s2d_workspace(*_s2d_args(spec))))


def _small_weights(spec: "ConvSpec", w):
    """W2[k][(r, s, c)] (bf16, columns padded to a multiple of 64) from [1][C_b][R][S][b_c][64]."""
    torch = require_cuda()
    rsc = spec.r * spec.s * spec.c
    ld = -(-rsc // 64) * 64
    w2 = torch.zeros((64, ld), dtype=torch.bfloat16, device="cuda")
    w2[:, :rsc] = w.permute(0, 2, 3, 1, 4, 5).reshape(rsc, 64).t()
    return w2, rsc, ld


def _small_im2col(spec: "ConvSpec", x, ld: int):
    torch = require_cuda()
    pix = spec.n * spec.out_h * spec.out_w
    col = torch.empty((pix, ld), dtype=torch.bfloat16, device="cuda")
    _lib.check(_lib.load().brk_conv_im2col(x.data_ptr(), col.data_ptr(), spec.n, spec.c, spec.h, spec.w, spec.r,
                                           spec.s, spec.stride, spec.pad_h, spec.pad_w, spec.b_c, ld, stream_ptr()),
               LayoutError)
    return col


def _geom(spec: "ConvSpec"):
    return (spec.n, spec.c, spec.k, spec.h, spec.w, spec.r, spec.s, spec.stride, spec.pad_h, spec.pad_w)


_WS: dict = {}


def _workspace(nbytes: int):
    torch = require_cuda()
    dev = torch.cuda.current_device()
    buf = _WS.get(dev)
    if nbytes and (buf is None or buf.numel() < nbytes):
        buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        _WS[dev] = buf
    return buf


def engine_plan(spec: "ConvSpec", pass_: int):
    """(pair, BN, splits) the engine uses for pass 0 fwd / 1 bwd-data / 2 upd (diagnostic)."""
    import ctypes
    out = (ctypes.c_int * 3)()
    _lib.check(_lib.load().brk_conv_plan(pass_, *_geom(spec), out), LayoutError)
    return tuple(out)


def _grid(*ranges, device="cuda"):
    """Flattened index grids (row-major over the given extents) as int64 device tensors."""
    torch = require_cuda()
    axes = [torch.arange(r, device=device, dtype=torch.int64) for r in ranges]
    mesh = torch.meshgrid(*axes, indexing="ij")
    return [m.reshape(-1) for m in mesh]


def conv2d_forward(spec: ConvSpec, inp: BlockedTensor, wgt: BlockedTensor, strategy: ParallelStrategy | None = None,
                   collapse: bool | None = None, tile_force=None, precision: str | None = None,
                   engine: bool | None = None) -> BlockedTensor:
    """O[N][K_b][P][Q][b_k] from I[N][C_b][H][W][b_c] and W[K_b][C_b][R][S][b_c][b_k] (cnn.py:201-334).

    ``engine``: None = the implicit-GEMM engine when the shape allows it,
    True = require it, False = the grouped BRGEMM path.
    """
    spec.validate()
    _check_layouts(spec, inp, wgt)
    if strategy is not None and strategy.workers < 1:
        raise ValueError(f"workers must be >= 1, got {strategy.workers}")
    torch = require_cuda()
    host = not inp.on_device
    prec, dt = _dtype(precision, inp, wgt)
    if _s2d_ok(spec, dt, engine):
        x, w = _stage(inp, dt), _stage(wgt, dt)
        out = torch.empty((spec.n, spec.k_blocks, spec.out_h, spec.out_w, 64), dtype=dt, device="cuda")
        ws = _s2d_workspace(spec)
        _lib.check(_lib.load().brk_conv_s2d_fwd(x.data_ptr(), w.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(),
                                                *_s2d_args(spec), stream_ptr()), LayoutError)
        res = BlockedTensor(out, n_outer=4, logical_dims={"n": 0, "k": (1, 4), "p": 2, "q": 3})
        return res.to("cpu") if host else res
    if _small_ok(spec, dt, engine):
        from ._dense import gemm
        x, w = _stage(inp, dt), _stage(wgt, dt)
        w2, rsc, _ = _small_weights(spec, w)
        col = _small_im2col(spec, x, -(-rsc // 8) * 8)  # dense rows: the GEMM reads K = R*S*C
        out = torch.empty((spec.n, 1, spec.out_h, spec.out_w, 64), dtype=dt, device="cuda")
        gemm(col[:, :rsc], w2[:, :rsc], out.view(-1, 64))
        res = BlockedTensor(out, n_outer=4, logical_dims={"n": 0, "k": (1, 4), "p": 2, "q": 3})
        return res.to("cpu") if host else res
    if _engine_ok(spec, dt, "fwd", engine):
        x, w = _stage(inp, dt), _stage(wgt, dt)
        out = torch.empty((spec.n, spec.k_blocks, spec.out_h, spec.out_w, spec.b_k), dtype=dt, device="cuda")
        code = _lib.BRK_BF16 if dt == torch.bfloat16 else _lib.BRK_F32
        _lib.check(_lib.load().brk_conv_fwd(x.data_ptr(), w.data_ptr(), None, out.data_ptr(), *_geom(spec), 64, 64,
                                            0, code, stream_ptr()), LayoutError)
        res = BlockedTensor(out, n_outer=4, logical_dims={"n": 0, "k": (1, 4), "p": 2, "q": 3})
        return res.to("cpu") if host else res
    x = _pad_device(_stage(inp, dt), spec.pad_h, spec.pad_w)
    w = _stage(wgt, dt)
    p_, q_ = spec.out_h, spec.out_w
    n, kb_n, cb_n, r_n, s_n = spec.n, spec.k_blocks, spec.c_blocks, spec.r, spec.s
    b_c, b_k, st = spec.b_c, spec.b_k, spec.stride
    hp, wp = spec.h + 2 * spec.pad_h, spec.w + 2 * spec.pad_w
    out = torch.empty((n, kb_n, p_, q_, b_k), dtype=dt, device="cuda")
    # jobs (img, kb, oj); entries (cb, r, s)
    ji, jk, jo = _grid(n, kb_n, p_)
    ec, er, es = _grid(cb_n, r_n, s_n)
    a_off = (((jk[:, None] * cb_n + ec[None, :]) * r_n + er[None, :]) * s_n + es[None, :]) * (b_c * b_k)
    b_off = (((ji[:, None] * cb_n + ec[None, :]) * hp + (jo[:, None] * st + er[None, :])) * wp + es[None, :]) * b_c
    c_off = ((ji * kb_n + jk) * p_ + jo) * (q_ * b_k)
    run_grouped(a_ptrs=addr_table(w, a_off.reshape(-1)), b_ptrs=addr_table(x, b_off.reshape(-1)),
                c_ptrs=addr_table(out, c_off), m=b_k, n=q_, k=b_c, batch=cb_n * r_n * s_n,
                a_sk=b_k, a_sm=1, b_sn=st * b_c, b_sk=1, ldc=b_k,
                in_bf16=dt == torch.bfloat16, out_bf16=dt == torch.bfloat16, precision=prec, exc=LayoutError)
    res = BlockedTensor(out, n_outer=4, logical_dims={"n": 0, "k": (1, 4), "p": 2, "q": 3})
    return res.to("cpu") if host else res


def conv2d_backward_data(spec: ConvSpec, dout: BlockedTensor, wgt: BlockedTensor,
                         precision: str | None = None, engine: bool | None = None) -> BlockedTensor:
    """dI[N][C_b][H][W][b_c] from dO[N][K_b][P][Q][b_k] (north star; restated in oracle/).

    Dual convolution of dO (dilated by the stride, padded by R-1-pad) with the
    flipped, C<->K-swapped filter; unpadded 1x1 stride-s: a 1x1 GEMM scattered
    to the strided input pixels (other pixels receive no gradient).
    """
    spec.validate()
    want = {"n": spec.n, "k": spec.k, "p": spec.out_h, "q": spec.out_w}
    if dout.logical_shape() != want or dout.inner_shape != (spec.b_k,):
        raise LayoutError(f"dout layout {dout.logical_shape()}/{dout.inner_shape} does not match spec")
    want_w = {"k": spec.k, "c": spec.c, "r": spec.r, "s": spec.s}
    if wgt.logical_shape() != want_w or wgt.inner_shape != (spec.b_c, spec.b_k):
        raise LayoutError("weight layout does not match spec")
    torch = require_cuda()
    host = not dout.on_device
    prec, dt = _dtype(precision, dout, wgt)
    do = _stage(dout, dt)
    w = _stage(wgt, dt)
    if _s2d_ok(spec, dt, engine):
        din = torch.empty((spec.n, spec.c_blocks, spec.h, spec.w, spec.b_c), dtype=dt, device="cuda")
        ws = _s2d_workspace(spec)
        _lib.check(_lib.load().brk_conv_s2d_bwd_data(do.data_ptr(), w.data_ptr(), din.data_ptr(), ws.data_ptr(),
                                                     ws.numel(), *_s2d_args(spec), stream_ptr()), LayoutError)
        res = BlockedTensor(din, n_outer=4, logical_dims={"n": 0, "c": (1, 4), "h": 2, "w": 3})
        return res.to("cpu") if host else res
    if _small_ok(spec, dt, engine):
        from ._dense import gemm
        w2, rsc, ld = _small_weights(spec, w)
        pix = spec.n * spec.out_h * spec.out_w
        dcol = torch.empty((pix, ld), dtype=dt, device="cuda")
        gemm(do.reshape(pix, 64), w2, dcol, b_t=True)  # dcol[pix][(r,s,c)] = dO[pix] . W[:, (r,s,c)]
        din = torch.empty((spec.n, spec.c_blocks, spec.h, spec.w, spec.b_c), dtype=dt, device="cuda")
        _lib.check(_lib.load().brk_conv_col2im(dcol.data_ptr(), din.data_ptr(), spec.n, spec.c, spec.h, spec.w,
                                               spec.r, spec.s, spec.stride, spec.pad_h, spec.pad_w, spec.b_c, ld,
                                               stream_ptr()), LayoutError)
        res = BlockedTensor(din, n_outer=4, logical_dims={"n": 0, "c": (1, 4), "h": 2, "w": 3})
        return res.to("cpu") if host else res
    if _engine_ok(spec, dt, "bwd", engine):
        din = torch.empty((spec.n, spec.c_blocks, spec.h, spec.w, spec.b_c), dtype=dt, device="cuda")
        code = _lib.BRK_BF16 if dt == torch.bfloat16 else _lib.BRK_F32
        _lib.check(_lib.load().brk_conv_bwd_data(do.data_ptr(), w.data_ptr(), din.data_ptr(), *_geom(spec), 64, 64,
                                                 code, stream_ptr()), LayoutError)
        res = BlockedTensor(din, n_outer=4, logical_dims={"n": 0, "c": (1, 4), "h": 2, "w": 3})
        return res.to("cpu") if host else res
    n, kb_n, cb_n, r_n, s_n = spec.n, spec.k_blocks, spec.c_blocks, spec.r, spec.s
    b_c, b_k, st = spec.b_c, spec.b_k, spec.stride
    p_, q_ = spec.out_h, spec.out_w
    h, wd = spec.h, spec.w
    din = torch.zeros((n, cb_n, h, wd, b_c), dtype=dt, device="cuda")
    in_bf16 = dt == torch.bfloat16
    if st == 1 or r_n > 1 or s_n > 1 or spec.pad_h or spec.pad_w:
        # dual convolution: dO dilated by the stride (zero insertion; a no-op for
        # stride 1), padded by R-1-pad on the leading side and by
        # R-1-pad + ((H + 2 pad - R) mod stride) on the trailing side, convolved
        # at stride 1 with the flipped, C<->K-swapped filter -> exactly H x W.
        ph, pw = r_n - 1 - spec.pad_h, s_n - 1 - spec.pad_w
        if ph < 0 or pw < 0:
            raise LayoutError("backward-data needs pad <= filter-1")
        pd, qd = (p_ - 1) * st + 1, (q_ - 1) * st + 1
        hp, wp = h + r_n - 1, wd + s_n - 1
        if st == 1 and hp == p_ + 2 * ph and wp == q_ + 2 * pw:
            dop = _pad_device(do, ph, pw)
        else:
            dop = torch.zeros((n, kb_n, hp, wp, b_k), dtype=do.dtype, device="cuda")
            dop[:, :, ph:ph + pd:st, pw:pw + qd:st] = do
        # dual conv output extent must equal the input extent
        if hp - r_n + 1 != h or wp - s_n + 1 != wd:
            raise LayoutError("backward-data: dual convolution does not reproduce the input extent")
        ji, jc, jh = _grid(n, cb_n, h)
        ek, er, es = _grid(kb_n, r_n, s_n)
        # A_i = W[kb][cb][R-1-r][S-1-s] viewed (k = b_k rows, m = b_c cols): a_sk = 1, a_sm = b_k
        a_off = (((ek[None, :] * cb_n + jc[:, None]) * r_n + (r_n - 1 - er[None, :])) * s_n
                 + (s_n - 1 - es[None, :])) * (b_c * b_k)
        b_off = (((ji[:, None] * kb_n + ek[None, :]) * hp + (jh[:, None] + er[None, :])) * wp + es[None, :]) * b_k
        c_off = ((ji * cb_n + jc) * h + jh) * (wd * b_c)
        run_grouped(a_ptrs=addr_table(w, a_off.reshape(-1)), b_ptrs=addr_table(dop, b_off.reshape(-1)),
                    c_ptrs=addr_table(din, c_off), m=b_c, n=wd, k=b_k, batch=kb_n * r_n * s_n,
                    a_sk=1, a_sm=b_k, b_sn=b_k, b_sk=1, ldc=b_c,
                    in_bf16=in_bf16, out_bf16=in_bf16, precision=prec, exc=LayoutError)
    else:
        # unpadded strided 1x1: dI[n][cb][oj*st][oi*st] = sum_kb dO[n][kb][oj][oi] W[kb][cb]^T,
        # the other input pixels receive no gradient (din is zero-initialised)
        ji, jc, jo = _grid(n, cb_n, p_)
        ek = torch.arange(kb_n, device="cuda", dtype=torch.int64)
        a_off = (ek[None, :] * cb_n + jc[:, None]) * (b_c * b_k)
        b_off = ((ji[:, None] * kb_n + ek[None, :]) * p_ + jo[:, None]) * (q_ * b_k)
        c_off = ((ji * cb_n + jc) * h + jo * st) * (wd * b_c)
        run_grouped(a_ptrs=addr_table(w, a_off.reshape(-1)), b_ptrs=addr_table(do, b_off.reshape(-1)),
                    c_ptrs=addr_table(din, c_off), m=b_c, n=q_, k=b_k, batch=kb_n,
                    a_sk=1, a_sm=b_k, b_sn=b_k, b_sk=1, ldc=st * b_c,
                    in_bf16=in_bf16, out_bf16=in_bf16, precision=prec, exc=LayoutError)
    res = BlockedTensor(din, n_outer=4, logical_dims={"n": 0, "c": (1, 4), "h": 2, "w": 3})
    return res.to("cpu") if host else res


def conv2d_weight_update(spec: ConvSpec, inp: BlockedTensor, dout: BlockedTensor,
                         precision: str | None = None, engine: bool | None = None) -> BlockedTensor:
    """dW[K_b][C_b][R][S][b_c][b_k] (fp32) = sum over (n, p, q) of dO x I_pad (north star)."""
    spec.validate()
    want_in = {"n": spec.n, "c": spec.c, "h": spec.h, "w": spec.w}
    if inp.logical_shape() != want_in or inp.inner_shape != (spec.b_c,):
        raise LayoutError("input layout does not match spec")
    want = {"n": spec.n, "k": spec.k, "p": spec.out_h, "q": spec.out_w}
    if dout.logical_shape() != want or dout.inner_shape != (spec.b_k,):
        raise LayoutError("dout layout does not match spec")
    torch = require_cuda()
    host = not inp.on_device
    prec, dt = _dtype(precision, inp, dout)
    if _s2d_ok(spec, dt, engine):
        x, do = _stage(inp, dt), _stage(dout, dt)
        dw = torch.empty((spec.k_blocks, spec.c_blocks, spec.r, spec.s, spec.b_c, spec.b_k), dtype=torch.float32,
                         device="cuda")
        ws = _s2d_workspace(spec)
        _lib.check(_lib.load().brk_conv_s2d_upd(x.data_ptr(), do.data_ptr(), dw.data_ptr(), ws.data_ptr(), ws.numel(),
                                                *_s2d_args(spec), stream_ptr()), LayoutError)
        res = BlockedTensor(dw, n_outer=4, logical_dims={"k": (0, 5), "c": (1, 4), "r": 2, "s": 3})
        return res.to("cpu") if host else res
    if _small_ok(spec, dt, engine):
        from ._dense import gemm
        x, do = _stage(inp, dt), _stage(dout, dt)
        rsc = spec.r * spec.s * spec.c
        col = _small_im2col(spec, x, -(-rsc // 8) * 8)
        pix = spec.n * spec.out_h * spec.out_w
        dwt = torch.empty((rsc, 64), dtype=torch.float32, device="cuda")
        gemm(col[:, :rsc], do.reshape(pix, 64), dwt, a_t=True, b_t=True)  # reduction over all pixels in TMEM
        dw = (dwt.reshape(spec.r, spec.s, spec.c_blocks, spec.b_c, 64).permute(2, 0, 1, 3, 4)
              .unsqueeze(0).contiguous())
        res = BlockedTensor(dw, n_outer=4, logical_dims={"k": (0, 5), "c": (1, 4), "r": 2, "s": 3})
        return res.to("cpu") if host else res
    if _engine_ok(spec, dt, "upd", engine):
        x, do = _stage(inp, dt), _stage(dout, dt)
        dw = torch.empty((spec.k_blocks, spec.c_blocks, spec.r, spec.s, spec.b_c, spec.b_k), dtype=torch.float32,
                         device="cuda")
        lib = _lib.load()
        nbytes = lib.brk_conv_upd_workspace(*_geom(spec))
        ws = _workspace(nbytes)
        _lib.check(lib.brk_conv_upd(x.data_ptr(), do.data_ptr(), dw.data_ptr(), None, 0.0,
                                    ws.data_ptr() if nbytes else None, nbytes, *_geom(spec), 64, 64,
                                    _lib.BRK_BF16 if dt == torch.bfloat16 else _lib.BRK_F32, stream_ptr()),
                   LayoutError)
        res = BlockedTensor(dw, n_outer=4, logical_dims={"k": (0, 5), "c": (1, 4), "r": 2, "s": 3})
        return res.to("cpu") if host else res
    x = _pad_device(_stage(inp, dt), spec.pad_h, spec.pad_w)
    do = _stage(dout, dt)
    n, kb_n, cb_n, r_n, s_n = spec.n, spec.k_blocks, spec.c_blocks, spec.r, spec.s
    b_c, b_k, st = spec.b_c, spec.b_k, spec.stride
    p_, q_ = spec.out_h, spec.out_w
    hp, wp = spec.h + 2 * spec.pad_h, spec.w + 2 * spec.pad_w
    dw = torch.empty((kb_n, cb_n, r_n, s_n, b_c, b_k), dtype=torch.float32, device="cuda")
    jk, jc, jr, js = _grid(kb_n, cb_n, r_n, s_n)
    ei, eo = _grid(n, p_)
    # A_i = dO[img][kb][oj] (k = Q pixels, m = b_k); B_i = I_pad[img][cb][oj*st+r][s::st]^T (n = b_c, k = Q)
    a_off = ((ei[None, :] * kb_n + jk[:, None]) * p_ + eo[None, :]) * (q_ * b_k)
    b_off = (((ei[None, :] * cb_n + jc[:, None]) * hp + (eo[None, :] * st + jr[:, None])) * wp + js[:, None]) * b_c
    c_off = (((jk * cb_n + jc) * r_n + jr) * s_n + js) * (b_c * b_k)
    run_grouped(a_ptrs=addr_table(do, a_off.reshape(-1)), b_ptrs=addr_table(x, b_off.reshape(-1)),
                c_ptrs=addr_table(dw, c_off), m=b_k, n=b_c, k=q_, batch=n * p_,
                a_sk=b_k, a_sm=1, b_sn=1, b_sk=st * b_c, ldc=b_k,
                in_bf16=dt == torch.bfloat16, out_bf16=False, precision=prec, exc=LayoutError)
    res = BlockedTensor(dw, n_outer=4, logical_dims={"k": (0, 5), "c": (1, 4), "r": 2, "s": 3})
    return res.to("cpu") if host else res


__all__ = [
    "ConvSpec", "ParallelStrategy", "PixelCollapse", "StrategyKind", "choose_strategy", "collapse_pixels",
    "conv2d_forward", "conv2d_backward_data", "conv2d_weight_update", "engine_plan", "make_conv_output",
]
