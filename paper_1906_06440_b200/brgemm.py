"""Batch-reduce GEMM (BRGEMM) on B200 tensor cores — drop-in for ``brkernels.brgemm``.

Computes ``C = beta*C + alpha * sum_i A_i @ B_i`` with the reference storage
contract (reference ``pkg/src/brkernels/brgemm.py:1-24``):

* ``a_blocks[i]`` has shape ``(k, m)`` (m contiguous, row stride ``lda``),
* ``b_blocks[i]`` has shape ``(n, k)`` (k contiguous, row stride ``ldb``),
* ``c`` has shape ``(n, m)`` (m contiguous, row stride ``ldc``).

Arithmetic runs in ``libbrk_sm100.so`` (tcgen05.mma, accumulator resident in
TMEM across the whole batch).  Inputs may be NumPy arrays (uploaded, result
written back into ``c`` in place, as the reference mutates ``c``) or CUDA
``torch.Tensor`` views (zero-copy).  The tensor-core input precision is TF32
or BF16 with fp32 accumulation (``BrgemmSpec.precision`` or
:func:`set_default_precision`); see DESIGN.md for the tolerance contract.

The CPU register-tile planner (``plan_tiles``/``TilePlan``) is kept for API
compatibility; the GPU picks its own tcgen05 tiles.
"""

from __future__ import annotations

import math
import os
from contextlib import contextmanager
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from ._device import is_torch, ptr_table, require_cuda, stream_ptr, upload

VLEN = 16
FMA_LATENCY = 5
REGISTER_BUDGET = 32
TILE_OVERRIDE_ENV = "BRGEMM_TILE_OVERRIDE"

PRECISIONS = ("tf32", "bf16")
_default_precision = "tf32"


class BrgemmError(ValueError):
    """Call-contract violation (operand lists, extents, strides or tile plans)."""


def set_default_precision(precision: str) -> None:
    """Select the tensor-core input type used when a spec does not name one."""
    global _default_precision
    if precision not in PRECISIONS:
        raise BrgemmError(f"precision must be one of {PRECISIONS}, got {precision!r}")
    _default_precision = precision


def get_default_precision() -> str:
    return _default_precision


@contextmanager
def precision(p: str):
    """Temporarily switch the default tensor-core input precision."""
    old = _default_precision
    set_default_precision(p)
    try:
        yield
    finally:
        set_default_precision(old)


@dataclass(frozen=True)
class BrgemmSpec:
    """Shape/scaling ledger of one BRGEMM call (reference brgemm.py:44-67).

    ``precision`` (new, optional) selects the tensor-core input type.
    """

    m: int
    n: int
    k: int
    batch: int
    alpha: float = 1.0
    beta: float = 1.0
    lda: int | None = None
    ldb: int | None = None
    ldc: int | None = None
    precision: str | None = None

    def __post_init__(self):
        for field_name in ("m", "n", "k", "batch"):
            value = getattr(self, field_name)
            if value < 0:
                raise BrgemmError(f"{field_name} must be >= 0, got {value}")
        if self.lda is not None and self.lda < self.m:
            raise BrgemmError(f"lda={self.lda} < m={self.m}")
        if self.ldb is not None and self.ldb < self.k:
            raise BrgemmError(f"ldb={self.ldb} < k={self.k}")
        if self.ldc is not None and self.ldc < self.m:
            raise BrgemmError(f"ldc={self.ldc} < m={self.m}")
        if self.precision is not None and self.precision not in PRECISIONS:
            raise BrgemmError(f"precision must be one of {PRECISIONS}, got {self.precision!r}")

    @property
    def resolved_precision(self) -> str:
        return self.precision or _default_precision


@dataclass(frozen=True)
class TilePlan:
    """CPU register-tile geometry (reference brgemm.py:70-91); API compatibility only."""

    m_b: int
    n_b: int
    vlen: int = VLEN
    fma_latency: int = FMA_LATENCY
    degraded: bool = False

    @property
    def accumulators(self) -> int:
        return self.n_b * math.ceil(self.m_b / self.vlen)

    @property
    def register_use(self) -> int:
        return self.accumulators + self.n_b + 1


def plan_tiles(m, n, vlen=VLEN, fma_latency=FMA_LATENCY, budget=REGISTER_BUDGET, force=None):
    """Register-tile search of the reference planner (brgemm.py:94-153).

    Objective, in priority order: most accumulators within the budget, m_b
    dividing m, larger m_b, larger n_b.  ``force`` is validated, not searched.
    """
    if m < 1 or n < 1:
        raise BrgemmError(f"extents must be >= 1, got m={m}, n={n}")
    if vlen < 1 or fma_latency < 1:
        raise BrgemmError("vlen and fma_latency must be >= 1")
    if budget < 3:
        raise BrgemmError(f"register budget must be >= 3, got {budget}")

    def finish(m_b, n_b):
        plan = TilePlan(m_b, n_b, vlen=vlen, fma_latency=fma_latency)
        return replace(plan, degraded=plan.accumulators < fma_latency)

    if force is not None:
        m_b, n_b = force
        if m_b < 1 or n_b < 1:
            raise BrgemmError(f"forced tile must be positive, got {force}")
        if m_b >= vlen and m_b % vlen:
            raise BrgemmError(f"forced m_b={m_b} is not a multiple of vlen={vlen}")
        plan = finish(m_b, n_b)
        if plan.register_use > budget:
            raise BrgemmError(
                f"forced tile {force} needs {plan.register_use} registers, budget {budget}"
            )
        return plan

    widths = [m] if m < vlen else list(range(vlen, (m // vlen) * vlen + 1, vlen))
    best_key, best = None, None
    for m_b in widths:
        vecs = -(-m_b // vlen)
        n_b = min(n, (budget - 1) // (vecs + 1))
        if n_b < 1:
            continue
        key = (n_b * vecs, m % m_b == 0, m_b, n_b)
        if best_key is None or key > best_key:
            best_key, best = key, (m_b, n_b)
    if best is None:
        best = (min(m, vlen), 1)
    return finish(*best)


def tile_override_from_env(env=None):
    """Parse BRGEMM_TILE_OVERRIDE="m_b,n_b" (reference brgemm.py:156-169)."""
    env = os.environ if env is None else env
    raw = env.get(TILE_OVERRIDE_ENV)
    if not raw:
        return None
    try:
        m_b, n_b = (int(part) for part in raw.split(","))
    except (TypeError, ValueError):
        raise BrgemmError(
            f"{TILE_OVERRIDE_ENV} must be 'm_b,n_b' integers, got {raw!r}"
        ) from None
    return m_b, n_b


# ---------------------------------------------------------------------------
# validation (same contract and messages as reference brgemm.py:172-207)
# ---------------------------------------------------------------------------
def _shape(x):
    return tuple(x.shape)


def _row_stride(x):
    if is_torch(x):
        return x.stride(0)
    return x.strides[0] // x.itemsize


def _check_blocks(a_blocks, b_blocks, c, spec: BrgemmSpec) -> None:
    if len(a_blocks) != spec.batch or len(b_blocks) != spec.batch:
        raise BrgemmError(
            f"operand list lengths ({len(a_blocks)}, {len(b_blocks)}) do not match batch={spec.batch}"
        )
    if _shape(c) != (spec.n, spec.m):
        raise BrgemmError(f"c has shape {_shape(c)}, expected {(spec.n, spec.m)}")
    for i, (a, b) in enumerate(zip(a_blocks, b_blocks)):
        if _shape(a) != (spec.k, spec.m):
            raise BrgemmError(f"a_blocks[{i}] has shape {_shape(a)}, expected {(spec.k, spec.m)}")
        if _shape(b) != (spec.n, spec.k):
            raise BrgemmError(f"b_blocks[{i}] has shape {_shape(b)}, expected {(spec.n, spec.k)}")
    if spec.lda is not None and spec.k > 1:
        if any(_row_stride(a) != spec.lda for a in a_blocks):
            raise BrgemmError(f"a block row stride != lda={spec.lda}")
    if spec.ldb is not None and spec.n > 1:
        if any(_row_stride(b) != spec.ldb for b in b_blocks):
            raise BrgemmError(f"b block row stride != ldb={spec.ldb}")
    if spec.ldc is not None and spec.n > 1 and _row_stride(c) != spec.ldc:
        raise BrgemmError(f"c row stride != ldc={spec.ldc}")


def _validate_plan(plan: TilePlan) -> None:
    if plan.m_b < 1 or plan.n_b < 1:
        raise BrgemmError(f"invalid tile plan ({plan.m_b}, {plan.n_b})")
    if plan.m_b >= plan.vlen and plan.m_b % plan.vlen:
        raise BrgemmError(f"invalid tile plan: m_b={plan.m_b} not a multiple of vlen={plan.vlen}")


# ---------------------------------------------------------------------------
# native dispatch
# ---------------------------------------------------------------------------
def _codes(spec: BrgemmSpec, in_bf16: bool):
    prec = spec.resolved_precision
    if in_bf16 and prec == "tf32":
        prec = "bf16"  # bf16 storage can only feed the bf16 tensor-core path
    compute = _lib.BRK_COMPUTE_TF32 if prec == "tf32" else _lib.BRK_COMPUTE_BF16
    return compute, (_lib.BRK_BF16 if in_bf16 else _lib.BRK_F32)


def _torch_ld(blocks, fallback):
    lds = {blk.stride(0) for blk in blocks}
    for blk in blocks:
        if blk.dim() != 2 or (blk.shape[1] > 1 and blk.stride(1) != 1):
            raise BrgemmError("device blocks must be 2-D with unit inner stride")
    if len(lds) > 1:
        raise BrgemmError("device blocks of one list must share a row stride")
    return lds.pop() if lds else fallback


def _one_storage(ts):
    base = ts[0].untyped_storage().data_ptr()
    return all(t.untyped_storage().data_ptr() == base and t.dtype == ts[0].dtype for t in ts)


def _check_device_dtypes(operands, outputs) -> bool:
    """Device operands: every A/B block one dtype in {float32, bfloat16}, every C
    float32 or bfloat16, all on the GPU.  Returns whether the inputs are bf16."""
    torch = require_cuda()
    ok = (torch.float32, torch.bfloat16)
    in_dt = operands[0].dtype if operands else torch.float32
    for t in operands:
        if not is_torch(t) or not t.is_cuda:
            raise BrgemmError("device BRGEMM: every A/B block must be a CUDA tensor")
        if t.dtype != in_dt:
            raise BrgemmError(f"device BRGEMM: mixed operand dtypes ({in_dt} and {t.dtype})")
    if in_dt not in ok:
        raise BrgemmError(f"device BRGEMM: operand dtype {in_dt} (need float32 or bfloat16)")
    for t in outputs:
        if not is_torch(t) or not t.is_cuda:
            raise BrgemmError("device BRGEMM: C must be a CUDA tensor")
        if t.dtype not in ok or t.dtype != outputs[0].dtype:
            raise BrgemmError(f"device BRGEMM: C dtype {t.dtype} (need one of float32 / bfloat16)")
    return in_dt == torch.bfloat16


def _run_addr_torch(a_list, b_list, c_list, m, n, k, batch, alpha, beta, spec):
    """All operands are CUDA tensors; a_list/b_list are job-major flat lists."""
    torch = require_cuda()
    in_bf16 = _check_device_dtypes(a_list + b_list, c_list)
    out_bf16 = c_list[0].dtype == torch.bfloat16
    compute, in_code = _codes(spec, in_bf16)
    lda = _torch_ld(a_list, m) if a_list else m
    ldb = _torch_ld(b_list, k) if b_list else k
    ldc = _torch_ld(c_list, m)
    c_tab = ptr_table([t.data_ptr() for t in c_list])
    lib = _lib.load()
    esz = a_list[0].element_size() if a_list else 0
    a_tab = ptr_table([t.data_ptr() for t in a_list]) if a_list else None
    b_tab = ptr_table([t.data_ptr() for t in b_list]) if b_list else None
    if a_list and b_list and _one_storage(a_list) and _one_storage(b_list):
        # blocks carved from one allocation per operand (the common case): register the two
        # allocations as views — the kernel turns each entry's pointers into view coordinates
        # and fetches in-bounds blocks with TMA (no host-side offset tables)
        sa, sb = a_list[0].untyped_storage(), b_list[0].untyped_storage()
        rc = lib.brk_brgemm_addr_views(
            a_tab.data_ptr(), b_tab.data_ptr(), c_tab.data_ptr(), sa.data_ptr(), sa.nbytes() // esz,
            sb.data_ptr(), sb.nbytes() // esz, len(c_list), m, n, k, batch, lda, ldb, ldc, float(alpha),
            float(beta), in_code, _lib.BRK_BF16 if out_bf16 else _lib.BRK_F32, compute, stream_ptr(),
        )
        _lib.check(rc, BrgemmError)
        return
    rc = lib.brk_brgemm_addr(
        a_tab.data_ptr() if a_tab is not None else None,
        b_tab.data_ptr() if b_tab is not None else None,
        c_tab.data_ptr(), len(c_list), m, n, k, batch, lda, ldb, ldc,
        float(alpha), float(beta), in_code,
        _lib.BRK_BF16 if out_bf16 else _lib.BRK_F32, compute, stream_ptr(),
    )
    _lib.check(rc, BrgemmError)


def _run_addr_numpy(a_blocks, b_blocks, c, spec, alpha, beta, jobs=1):
    """Upload packed copies of the host blocks, run the address variant, write c back."""
    torch = require_cuda()
    m, n, k, batch = spec.m, spec.n, spec.k, spec.batch
    dev_c = upload(np.asarray(c, dtype=np.float32).reshape(jobs, n, m))
    c_list = [dev_c[j] for j in range(jobs)]
    if batch and k:
        dev_a = upload(np.stack([np.asarray(a, dtype=np.float32) for a in a_blocks]))
        dev_b = upload(np.stack([np.asarray(b, dtype=np.float32) for b in b_blocks]))
        a_list = [dev_a[i] for i in range(dev_a.shape[0])]
        b_list = [dev_b[i] for i in range(dev_b.shape[0])]
    else:
        a_list, b_list = [], []
        batch = 0 if not k else batch
    if k == 0 and spec.batch:
        # (n,0)@(0,m) contributes exact zeros: run as an empty batch.
        batch = 0
    _run_addr_torch(a_list, b_list, c_list, m, n, k, batch, alpha, beta, spec)
    return dev_c.cpu().numpy()


def brgemm(a_blocks, b_blocks, c, spec: BrgemmSpec, plan: TilePlan | None = None):
    """Batch-reduce GEMM over address-designated blocks (reference brgemm.py:260-293).

    One output block, one tcgen05 accumulation chain across the whole batch,
    one store.  ``c`` is updated in place and returned.
    """
    if plan is None:
        plan = plan_tiles(max(spec.m, 1), max(spec.n, 1))
    _validate_plan(plan)
    _check_blocks(a_blocks, b_blocks, c, spec)
    if spec.m == 0 or spec.n == 0:
        return c
    batch = spec.batch if spec.alpha != 0.0 else 0
    if is_torch(c):
        if batch == 0 or spec.k == 0:
            _run_addr_torch([], [], [c], spec.m, spec.n, spec.k, 0, spec.alpha, spec.beta, spec)
        else:
            _run_addr_torch(list(a_blocks), list(b_blocks), [c], spec.m, spec.n, spec.k, batch,
                            spec.alpha, spec.beta, spec)
        return c
    if batch == 0:
        a_blocks, b_blocks = [], []
    out = _run_addr_numpy(a_blocks, b_blocks, c, replace(spec, batch=batch), spec.alpha, spec.beta)
    c[...] = out.reshape(c.shape)
    return c


def brgemm_accumulate(a_blocks, b_blocks, acc, spec: BrgemmSpec, plan: TilePlan | None = None):
    """acc += sum_i A_i @ B_i into a caller-owned float64 (n, m) buffer (brgemm.py:240-257).

    The tensor cores produce the fp32 batch sum in TMEM; it is added to the
    caller's float64 buffer once.
    """
    if plan is None:
        plan = plan_tiles(max(spec.m, 1), max(spec.n, 1))
    _validate_plan(plan)
    _check_blocks(a_blocks, b_blocks, acc, spec)
    if getattr(acc, "dtype", None) != np.float64:
        raise BrgemmError(f"accumulator must be float64, got {getattr(acc, 'dtype', None)}")
    if spec.m and spec.n and spec.batch:
        part = np.zeros((spec.n, spec.m), np.float32)
        part = _run_addr_numpy(a_blocks, b_blocks, part,
                               replace(spec, alpha=1.0, beta=0.0, lda=None, ldb=None, ldc=None),
                               1.0, 0.0)
        acc += part.reshape(spec.n, spec.m)
    return acc


def _flat_size(x):
    return int(x.numel()) if is_torch(x) else int(np.size(x))


def brgemm_strided(a_base, b_base, stride_a: int, stride_b: int, c, spec: BrgemmSpec,
                   plan: TilePlan | None = None):
    """Blocks at fixed element strides in flat buffers (reference brgemm.py:296-337).

    ``A_i`` starts at element ``i*stride_a`` of the flattened ``a_base`` (ditto B).
    Runs the native stride variant directly on the flat buffers.
    """
    if stride_a < 0 or stride_b < 0:
        raise BrgemmError("strides must be >= 0")
    a_span, b_span = spec.k * spec.m, spec.n * spec.k
    if spec.batch > 0:
        need_a = (spec.batch - 1) * stride_a + a_span
        need_b = (spec.batch - 1) * stride_b + b_span
        if need_a > _flat_size(a_base):
            raise BrgemmError(
                f"stride_a={stride_a} with batch={spec.batch} overruns A ({need_a} > {_flat_size(a_base)})"
            )
        if need_b > _flat_size(b_base):
            raise BrgemmError(
                f"stride_b={stride_b} with batch={spec.batch} overruns B ({need_b} > {_flat_size(b_base)})"
            )
    if plan is None:
        plan = plan_tiles(max(spec.m, 1), max(spec.n, 1))
    _validate_plan(plan)
    if _shape(c) != (spec.n, spec.m):
        raise BrgemmError(f"c has shape {_shape(c)}, expected {(spec.n, spec.m)}")
    if spec.m == 0 or spec.n == 0:
        return c
    torch = require_cuda()
    batch = spec.batch if (spec.alpha != 0.0 and spec.k > 0) else 0
    host = not is_torch(c)
    if host:
        dev_a = upload(np.ravel(np.asarray(a_base, dtype=np.float32))) if batch else None
        dev_b = upload(np.ravel(np.asarray(b_base, dtype=np.float32))) if batch else None
        dev_c = upload(np.asarray(c, dtype=np.float32))
    else:
        dev_a = a_base.reshape(-1) if batch else None
        dev_b = b_base.reshape(-1) if batch else None
        dev_c = c
        if not dev_c.is_contiguous():
            raise BrgemmError("device c must be contiguous for the stride variant")
    in_bf16 = _check_device_dtypes([t for t in (dev_a, dev_b) if t is not None], [dev_c])
    compute, in_code = _codes(spec, in_bf16)
    lib = _lib.load()
    rc = lib.brk_brgemm_stride(
        dev_a.data_ptr() if dev_a is not None else None,
        dev_b.data_ptr() if dev_b is not None else None,
        int(stride_a), int(stride_b), dev_c.data_ptr(), 1, 0, 0, 0,
        spec.m, spec.n, spec.k, batch, spec.m, spec.k, spec.m,
        float(spec.alpha), float(spec.beta), in_code,
        _lib.BRK_BF16 if dev_c.dtype == torch.bfloat16 else _lib.BRK_F32, compute, stream_ptr(),
    )
    _lib.check(rc, BrgemmError)
    if host:
        c[...] = dev_c.cpu().numpy()
    return c


def brgemm_offset(a_base, b_base, a_offsets, b_offsets, c, spec: BrgemmSpec,
                  plan: TilePlan | None = None):
    """Offset variant (north star): ``A_i = a_base.flat[a_offsets[i]:]`` viewed (k, m).

    Blocks are packed (row strides m and k).  Equivalent to :func:`brgemm` on the
    corresponding address list; runs the native offset variant.
    """
    a_offsets = [int(o) for o in a_offsets]
    b_offsets = [int(o) for o in b_offsets]
    if len(a_offsets) != spec.batch or len(b_offsets) != spec.batch:
        raise BrgemmError(
            f"offset list lengths ({len(a_offsets)}, {len(b_offsets)}) do not match batch={spec.batch}"
        )
    a_span, b_span = spec.k * spec.m, spec.n * spec.k
    for name, offs, span, base in (("A", a_offsets, a_span, a_base), ("B", b_offsets, b_span, b_base)):
        for o in offs:
            if o < 0 or o + span > _flat_size(base):
                raise BrgemmError(f"offset {o} overruns {name} ({o + span} > {_flat_size(base)})")
    if plan is None:
        plan = plan_tiles(max(spec.m, 1), max(spec.n, 1))
    _validate_plan(plan)
    if _shape(c) != (spec.n, spec.m):
        raise BrgemmError(f"c has shape {_shape(c)}, expected {(spec.n, spec.m)}")
    if spec.m == 0 or spec.n == 0:
        return c
    torch = require_cuda()
    batch = spec.batch if (spec.alpha != 0.0 and spec.k > 0) else 0
    host = not is_torch(c)
    if host:
        dev_a = upload(np.ravel(np.asarray(a_base, dtype=np.float32)))
        dev_b = upload(np.ravel(np.asarray(b_base, dtype=np.float32)))
        dev_c = upload(np.asarray(c, dtype=np.float32))
    else:
        dev_a, dev_b, dev_c = a_base.reshape(-1), b_base.reshape(-1), c
    c_tab = ptr_table([dev_c.data_ptr()])
    a_off = torch.tensor(a_offsets or [0], dtype=torch.int64, device="cuda")
    b_off = torch.tensor(b_offsets or [0], dtype=torch.int64, device="cuda")
    compute, in_code = _codes(spec, _check_device_dtypes([dev_a, dev_b], [dev_c]))
    lib = _lib.load()
    rc = lib.brk_brgemm_offs(
        dev_a.data_ptr(), dev_b.data_ptr(), a_off.data_ptr(), b_off.data_ptr(), c_tab.data_ptr(),
        1, spec.m, spec.n, spec.k, batch, spec.m, spec.k, _row_stride(dev_c),
        float(spec.alpha), float(spec.beta), in_code,
        _lib.BRK_BF16 if dev_c.dtype == torch.bfloat16 else _lib.BRK_F32, compute, stream_ptr(),
    )
    _lib.check(rc, BrgemmError)
    if host:
        c[...] = dev_c.cpu().numpy()
    return c


def batched_gemm(a_blocks, b_blocks, c_blocks, spec: BrgemmSpec, plan: TilePlan | None = None):
    """No-reduction baseline ``C_i = beta*C_i + alpha*A_i@B_i`` (reference brgemm.py:340-353).

    All pairs run in ONE grouped launch (one job per pair, batch 1 each).
    """
    if len(c_blocks) != spec.batch:
        raise BrgemmError(f"c_blocks has length {len(c_blocks)}, expected batch={spec.batch}")
    single = replace(spec, batch=1)
    for a, b, ci in zip(a_blocks, b_blocks, c_blocks):
        _check_blocks([a], [b], ci, single)
    if plan is not None:
        _validate_plan(plan)
    if spec.batch == 0 or spec.m == 0 or spec.n == 0:
        return c_blocks
    use_batch = 1 if (spec.alpha != 0.0 and spec.k > 0) else 0
    if is_torch(c_blocks[0]):
        _run_addr_torch(list(a_blocks) if use_batch else [], list(b_blocks) if use_batch else [],
                        list(c_blocks), spec.m, spec.n, spec.k, use_batch, spec.alpha, spec.beta, spec)
        return c_blocks
    stacked_c = np.stack([np.asarray(ci, dtype=np.float32) for ci in c_blocks])
    out = _run_addr_numpy(a_blocks if use_batch else [], b_blocks if use_batch else [], stacked_c,
                          replace(spec, batch=use_batch), spec.alpha, spec.beta, jobs=spec.batch)
    out = out.reshape(spec.batch, spec.n, spec.m)
    for j, ci in enumerate(c_blocks):
        ci[...] = out[j]
    return c_blocks
