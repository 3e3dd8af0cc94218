"""Device plumbing shared by the operator modules: CUDA presence, streams, uploads.

PyTorch is used only for device memory, streams and host<->device copies; all
arithmetic on the product path runs in libbrk_sm100.so.
"""

from __future__ import annotations

import numpy as np

from ._lib import BrkNativeError, load

try:  # torch is the plumbing; importing it is mandatory on the product path
    import torch
except ImportError:  # pragma: no cover
    torch = None


def require_cuda():
    """Return the torch module after checking a CUDA device and the native library."""
    if torch is None:
        raise BrkNativeError("PyTorch is required for device memory; it is not importable")
    if not torch.cuda.is_available():
        raise BrkNativeError(
            "no CUDA device visible: the B200 path has no CPU fallback "
            "(run the oracle in oracle/ for CPU checks)"
        )
    load()
    return torch


def is_torch(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def stream_ptr() -> int:
    return int(torch.cuda.current_stream().cuda_stream)


def upload(arr: np.ndarray, dtype=None):
    """Host numpy array -> contiguous device tensor (optionally cast on device)."""
    t = torch.from_numpy(np.ascontiguousarray(arr)).to("cuda", non_blocking=False)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t


def ptr_table(ptrs) -> "torch.Tensor":
    """Device int64 table of raw addresses (the address-variant batch list)."""
    return torch.tensor(list(ptrs), dtype=torch.int64, device="cuda")
