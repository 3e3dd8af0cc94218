"""Launch helper for the grouped batch-list BRGEMM (``brk_brgemm_grouped``).

The drivers (fc / lstm / cnn) describe a pass as a set of output blocks
("jobs"), each with a batch list of (A_i, B_i) block addresses — exactly the
pointer lists the reference builds per work item (``fc.py:139-160``,
``cnn.py:241-252``) — but as device tables, so one launch covers the pass.
Address tables are built with integer tensor arithmetic on the device
(``base + elem_size * offsets``); no values are touched on the host.
"""

from __future__ import annotations

import ctypes

from . import _lib
from ._device import require_cuda, stream_ptr


def addr_table(base, offsets_elems):
    """int64 device table of ``base.data_ptr() + itemsize * offsets``."""
    import torch

    return offsets_elems.to(torch.int64) * base.element_size() + base.data_ptr()


def run_grouped(*, a_ptrs, b_ptrs, c_ptrs, m, n, k, batch, a_sk, a_sm, b_sn, b_sk, ldc,
                in_bf16, out_bf16, precision, alpha=1.0, beta=0.0, bias=None, bias_offs=None,
                act=0, mask_ptrs=None, exc=ValueError):
    torch = require_cuda()
    compute = _lib.BRK_COMPUTE_TF32 if (precision == "tf32" and not in_bf16) else _lib.BRK_COMPUTE_BF16
    keep = [t for t in (a_ptrs, b_ptrs, c_ptrs, bias, bias_offs, mask_ptrs) if t is not None]
    for t in keep:
        if not t.is_cuda or not t.is_contiguous():
            raise exc("grouped BRGEMM tables must be contiguous CUDA tensors")
    d = _lib.GroupedDesc()
    d.n_jobs = int(c_ptrs.numel())
    d.m, d.n, d.k, d.batch = int(m), int(n), int(k), int(batch)
    d.a_sk, d.a_sm, d.b_sn, d.b_sk, d.ldc = int(a_sk), int(a_sm), int(b_sn), int(b_sk), int(ldc)
    d.alpha, d.beta = float(alpha), float(beta)
    d.in_dtype = _lib.BRK_BF16 if in_bf16 else _lib.BRK_F32
    d.out_dtype = _lib.BRK_BF16 if out_bf16 else _lib.BRK_F32
    d.compute = compute
    d.a_ptrs = a_ptrs.data_ptr() if a_ptrs is not None else None
    d.b_ptrs = b_ptrs.data_ptr() if b_ptrs is not None else None
    d.c_ptrs = c_ptrs.data_ptr()
    d.bias = bias.data_ptr() if bias is not None else None
    d.bias_offs = bias_offs.data_ptr() if bias_offs is not None else None
    d.act = int(act)
    d.mask_ptrs = mask_ptrs.data_ptr() if mask_ptrs is not None else None
    rc = _lib.load().brk_brgemm_grouped(ctypes.byref(d), stream_ptr())
    _lib.check(rc, exc)
    del torch
