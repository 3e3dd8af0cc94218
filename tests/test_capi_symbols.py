"""The C-ABI library loads without a GPU and exports every symbol include/brk.h declares."""

import ctypes
import re
from pathlib import Path

from paper_1906_06440_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "brk.h").read_text()
    return set(re.findall(r"BRK_API\s+[\w\s\*]+?\b(brk_\w+)\s*\(", text))


def test_header_declares_api():
    syms = declared_symbols()
    assert {"brk_brgemm_addr", "brk_brgemm_offs", "brk_brgemm_stride", "brk_brgemm_grouped",
            "brk_fc_fwd", "brk_fc_bwd_data", "brk_fc_upd", "brk_last_error"} <= syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in sorted(declared_symbols()) if not hasattr(lib, s)]
    assert not missing, f"declared but not exported: {missing}"


def test_binding_table_covers_header():
    assert declared_symbols() == set(_lib.SIGNATURES), (
        declared_symbols() ^ set(_lib.SIGNATURES))


def test_load_and_contract_errors_without_gpu():
    lib = _lib.load()
    assert lib.brk_version() >= 1
    # contract violations are reported before any device work
    rc = lib.brk_brgemm_stride(None, None, -1, 0, None, 1, 0, 0, 0, 4, 4, 4, 1, 4, 4, 4, 1.0, 0.0,
                               _lib.BRK_F32, _lib.BRK_F32, _lib.BRK_COMPUTE_TF32, None)
    assert rc == _lib.BRK_ERR_CONTRACT
    assert "stride" in _lib.last_error()
    rc = lib.brk_fc_fwd(None, None, None, None, 100, 64, 64, 64, 64, 64, 0, _lib.BRK_BF16, None)
    assert rc == _lib.BRK_ERR_CONTRACT
    rc = lib.brk_brgemm_addr(None, None, None, 1, 8, 8, 8, 1, 4, 8, 8, 1.0, 0.0, _lib.BRK_F32,
                             _lib.BRK_F32, _lib.BRK_COMPUTE_TF32, None)
    assert rc == _lib.BRK_ERR_CONTRACT and "leading" in _lib.last_error()


def test_cubin_is_sm100a_tcgen05():
    """The shipped library carries sm_100a SASS with tcgen05 MMA and TMA."""
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        return
    out = subprocess.run([cuobjdump, "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out or "UTCQMMA" in out
    assert "UTMALDG" in out
    assert "LDTM" in out
