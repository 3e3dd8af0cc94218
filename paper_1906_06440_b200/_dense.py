"""Dense row-major GEMM on the tcgen05 engine (``brk_gemm_dense`` bf16 /
``brk_gemm_dense_f32`` TF32, include/brk.h): device plumbing for the LSTM
drivers (input projection over all steps, backward-data, weight gradients) and
the small-channel conv path.  Operands are torch tensors on the device; the
product path has no fallback."""

from __future__ import annotations

from . import _lib
from ._device import require_cuda, stream_ptr
from .tensor import LayoutError

_WS: dict = {}


def _workspace(nbytes: int):
    torch = require_cuda()
    dev = torch.cuda.current_device()
    buf = _WS.get(dev)
    if nbytes and (buf is None or buf.numel() < nbytes):
        buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        _WS[dev] = buf
    return buf


def _operand(t, rows: int, k: int, transposed: bool):
    """(ptr, ld, kmajor) of a 2-d bf16 / fp32 operand holding a rows x k matrix, given
    as rows x k (``transposed`` False) or k x rows (True), row-major contiguous rows."""
    torch = require_cuda()
    if t.dtype not in (torch.bfloat16, torch.float32) or t.dim() != 2 or t.stride(1) != 1:
        raise LayoutError("gemm_dense operands must be 2-d bf16 or fp32 with unit inner stride")
    want = (k, rows) if transposed else (rows, k)
    if tuple(t.shape) != want:
        raise LayoutError(f"gemm_dense operand shape {tuple(t.shape)} != {want}")
    return t.data_ptr(), t.stride(0), 0 if transposed else 1


def gemm(a, b, out, *, a_t: bool = False, b_t: bool = False, bias=None, relu: bool = False, beta: float = 0.0,
         split: bool = True):
    """out[M][N] = a . b^T (+ bias, ReLU) (+ beta * out).

    ``a`` is M x K (or K x M with ``a_t``); ``b`` is N x K (or K x N with ``b_t``);
    ``out`` fp32 or bf16 M x N with unit inner stride."""
    torch = require_cuda()
    M, N = out.shape
    K = a.shape[0] if a_t else a.shape[1]
    if a.dtype != b.dtype:
        raise LayoutError(f"gemm_dense operands must share a dtype ({a.dtype} vs {b.dtype})")
    f32 = a.dtype == torch.float32
    if f32:  # TF32 tensor cores: round-to-nearest copies of the operands (fc.tf32_operand)
        from .fc import tf32_operand
        a, b = tf32_operand(a), tf32_operand(b)
    pa, lda, ka = _operand(a, M, K, a_t)
    pb, ldb, kb = _operand(b, N, K, b_t)
    if out.stride(1) != 1:
        raise LayoutError("gemm_dense output needs unit inner stride")
    lib = _lib.load()
    nbytes = lib.brk_gemm_dense_workspace(M, N, K) if split and out.dtype == torch.float32 else 0
    ws = _workspace(nbytes)
    fn = lib.brk_gemm_dense_f32 if f32 else lib.brk_gemm_dense
    rc = fn(pa, lda, ka, pb, ldb, kb, out.data_ptr(), out.stride(0),
                            1 if out.dtype == torch.bfloat16 else 0, M, N, K, 1.0, beta,
                            bias.data_ptr() if bias is not None else None, 1 if relu else 0,
                            ws.data_ptr() if nbytes else None, nbytes, stream_ptr())
    _lib.check(rc, LayoutError)
    return out
