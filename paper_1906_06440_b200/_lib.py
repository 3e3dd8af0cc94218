"""ctypes binding of the in-tree C-ABI library ``libbrk_sm100.so`` (include/brk.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, every compute entry point raises ``BrkNativeError``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_NAME = "libbrk_sm100.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

BRK_OK = 0
BRK_ERR_CONTRACT = 1
BRK_ERR_CUDA = 2

BRK_F32 = 0
BRK_BF16 = 1
BRK_COMPUTE_TF32 = 0
BRK_COMPUTE_BF16 = 1

_c_int = ctypes.c_int
_c_i64 = ctypes.c_int64
_c_f = ctypes.c_float
_vp = ctypes.c_void_p

# name -> (restype, argtypes); the single source of truth for the exports
# tests/test_capi_symbols.py checks against include/brk.h.
SIGNATURES: dict[str, tuple] = {
    "brk_last_error": (ctypes.c_char_p, []),
    "brk_version": (_c_int, []),
    "brk_launch_count": (ctypes.c_uint64, []),
    "brk_brgemm_addr": (
        _c_int,
        [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_i64, _c_i64, _c_i64,
         _c_f, _c_f, _c_int, _c_int, _c_int, _vp],
    ),
    "brk_brgemm_addr_views": (
        _c_int,
        [_vp, _vp, _vp, _vp, _c_i64, _vp, _c_i64, _c_int, _c_int, _c_int, _c_int, _c_int, _c_i64, _c_i64,
         _c_i64, _c_f, _c_f, _c_int, _c_int, _c_int, _vp],
    ),
    "brk_brgemm_grouped": (_c_int, [_vp, _vp]),
    "brk_fc_fwd": (_c_int, [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                            _c_int, _c_int, _vp]),
    "brk_fc_bwd_data": (_c_int, [_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                                 _c_int, _vp]),
    "brk_fc_upd": (_c_int, [_vp, _vp, _vp, _vp, _c_f, _vp, _c_int, _vp, _vp, _c_f, _vp, ctypes.c_size_t,
                            _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp]),
    "brk_fc_upd_workspace": (ctypes.c_size_t, [_c_int, _c_int, _c_int]),
    "brk_mlp_step": (_c_int, [_c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_f, _vp,
                              ctypes.c_size_t, _vp]),
    "brk_mlp_step_dt": (_c_int, [_c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_f, _vp,
                                 ctypes.c_size_t, _c_int, _vp]),
    "brk_mlp_step_workspace_bytes": (ctypes.c_size_t, [_c_int, _c_int, _c_int]),
    "brk_diag_set_timestamps": (None, [_vp]),
    "brk_lstm_fwd_step": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp]),
    "brk_lstm_bwd_step": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int,
                                   _vp]),
    "brk_lstm_recurrent_grad": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp]),
    "brk_diag_tmem_ld": (_c_int, [_c_int, _c_int, _vp, _vp]),
    "brk_diag_mma_rate": (_c_int, [_c_int, _c_int, _c_int, _c_int, _vp]),
    "brk_diag_tma_lanes": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp]),
    "brk_diag_mlp_schedule": (_c_int, [_c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp]),
    "brk_diag_tma_bw": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                                 ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double)]),
    "brk_fc_bias_grad": (_c_int, [_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_f, _vp]),
    "brk_fc_bias_grad_workspace": (ctypes.c_size_t, [_c_int]),
    "brk_fc_bias_grad_dt": (_c_int, [_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_f, _c_int,
                                     _vp]),
    "brk_colsum_blocked": (_c_int, [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp]),
    "brk_sgd_apply": (_c_int, [_vp, _vp, _c_f, _c_i64, _c_int, _vp]),
    "brk_layout_transform": (_c_int, [_vp, _vp, _c_int, _vp, _vp, _vp, _vp, _c_int, _c_int, _vp]),
    "brk_conv_fwd": (_c_int, [_vp, _vp, _vp, _vp] + [_c_int] * 14 + [_vp]),
    "brk_conv_bwd_data": (_c_int, [_vp, _vp, _vp] + [_c_int] * 13 + [_vp]),
    "brk_conv_upd": (_c_int, [_vp, _vp, _vp, _vp, _c_f, _vp, ctypes.c_size_t] + [_c_int] * 13 + [_vp]),
    "brk_conv_upd_workspace": (ctypes.c_size_t, [_c_int] * 10),
    "brk_conv_plan": (_c_int, [_c_int] * 11 + [ctypes.POINTER(_c_int)]),
    "brk_conv_im2col": (_c_int, [_vp, _vp] + [_c_int] * 10 + [_c_i64, _vp]),
    "brk_conv_col2im": (_c_int, [_vp, _vp] + [_c_int] * 10 + [_c_i64, _vp]),
    "brk_conv_s2d_shape": (_c_int, [_c_int] * 9 + [ctypes.POINTER(_c_int)]),
    "brk_conv_s2d_workspace": (ctypes.c_size_t, [_c_int] * 9),
    "brk_conv_s2d_unfold": (_c_int, [_vp, _vp] + [_c_int] * 8 + [_vp]),
    "brk_conv_s2d_fwd": (_c_int, [_vp, _vp, _vp, _vp, ctypes.c_size_t] + [_c_int] * 9 + [_vp]),
    "brk_conv_s2d_upd": (_c_int, [_vp, _vp, _vp, _vp, ctypes.c_size_t] + [_c_int] * 9 + [_vp]),
    "brk_conv_s2d_bwd_data": (_c_int, [_vp, _vp, _vp, _vp, ctypes.c_size_t] + [_c_int] * 9 + [_vp]),
    "brk_gemm_dense": (_c_int, [_vp, _c_i64, _c_int, _vp, _c_i64, _c_int, _vp, _c_i64, _c_int, _c_i64, _c_int,
                                _c_int, _c_f, _c_f, _vp, _c_int, _vp, ctypes.c_size_t, _vp]),
    "brk_gemm_dense_workspace": (ctypes.c_size_t, [_c_i64, _c_int, _c_int]),
    "brk_gemm_dense_f32": (_c_int, [_vp, _c_i64, _c_int, _vp, _c_i64, _c_int, _vp, _c_i64, _c_int, _c_i64, _c_int,
                                    _c_int, _c_f, _c_f, _vp, _c_int, _vp, ctypes.c_size_t, _vp]),
    "brk_round_tf32": (_c_int, [_vp, _vp, _c_i64, _vp]),
    "brk_lstm_seq_flags_bytes": (ctypes.c_size_t, [_c_int]),
    "brk_diag_lstm_timestamps": (None, [_vp]),
    "brk_lstm_seq_fwd": (_c_int, [_vp] * 8 + [_c_int, _c_int, _c_int, _vp]),
    "brk_lstm_seq_bwd": (_c_int, [_vp] * 8 + [_c_int, _c_int, _c_int, _vp]),
    "brk_brgemm_offs": (
        _c_int,
        [_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_i64, _c_i64, _c_i64,
         _c_f, _c_f, _c_int, _c_int, _c_int, _vp],
    ),
    "brk_brgemm_stride": (
        _c_int,
        [_vp, _vp, _c_i64, _c_i64, _vp, _c_int, _c_i64, _c_i64, _c_i64, _c_int, _c_int, _c_int,
         _c_int, _c_i64, _c_i64, _c_i64, _c_f, _c_f, _c_int, _c_int, _c_int, _vp],
    ),
}


class GroupedDesc(ctypes.Structure):
    """Mirror of ``brk_grouped_desc`` (include/brk.h)."""

    _fields_ = [
        ("n_jobs", _c_int), ("m", _c_int), ("n", _c_int), ("k", _c_int), ("batch", _c_int),
        ("a_sk", _c_i64), ("a_sm", _c_i64), ("b_sn", _c_i64), ("b_sk", _c_i64), ("ldc", _c_i64),
        ("alpha", _c_f), ("beta", _c_f),
        ("in_dtype", _c_int), ("out_dtype", _c_int), ("compute", _c_int),
        ("a_ptrs", _vp), ("b_ptrs", _vp), ("c_ptrs", _vp),
        ("bias", _vp), ("bias_offs", _vp), ("act", _c_int), ("mask_ptrs", _vp),
    ]


class BrkNativeError(RuntimeError):
    """The native library is missing, failed to load, or returned a CUDA error."""


_lib = None


def load(path: os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and return the C-ABI library; raise loudly if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # BRK_LIB: an alternative build of the same library (e.g. the diagnostics build
    # libbrk_sm100_diag.so with in-kernel timestamps, `make -C csrc diag`)
    p = Path(path) if path is not None else Path(os.environ.get("BRK_LIB", LIB_PATH))
    if not p.exists():
        raise BrkNativeError(
            f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(or `make -C paper_1906_06440_b200/csrc`). There is no CPU fallback."
        )
    try:
        lib = ctypes.CDLL(str(p))
    except OSError as exc:  # pragma: no cover - depends on the box
        raise BrkNativeError(f"failed to load {p}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def last_error() -> str:
    return load().brk_last_error().decode("utf-8", "replace")


def check(rc: int, contract_exc=ValueError) -> None:
    """Map a C-ABI return code to the reference's exception classes."""
    if rc == BRK_OK:
        return
    msg = last_error()
    if rc == BRK_ERR_CONTRACT:
        raise contract_exc(msg)
    raise BrkNativeError(msg)


def launch_count() -> int:
    return int(load().brk_launch_count())
