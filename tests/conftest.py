"""Shared test fixtures: repo on sys.path, the `gpu` marker, golden-vector loader,
and the parity-error log (every GPU parity check records its measured error;
the terminal summary prints the worst per check and, when ``gpurun_out/``
exists, the full table goes to ``gpurun_out/parity_errors.json``)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

GOLDEN = ROOT / "tests" / "golden"

# name -> list of (case, error, tolerance)
PARITY_LOG: dict = {}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libbrk_sm100.so")


def record_parity(name: str, case, err: float, tol: float) -> float:
    """Log one measured error (scale-relative unless the name says otherwise) and return it."""
    PARITY_LOG.setdefault(name, []).append((str(case), float(err), float(tol)))
    return err


def check_parity(name: str, case, err: float, tol: float) -> None:
    record_parity(name, case, err, tol)
    assert err <= tol, f"{name} {case}: error {err:.3e} > tolerance {tol:.1e}"


@pytest.fixture
def parity():
    return check_parity


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    if not PARITY_LOG:
        return
    tr = terminalreporter
    tr.section("parity errors (worst per check; scale-relative max|got-ref|/max|ref|)")
    rows = {}
    for name, vals in sorted(PARITY_LOG.items()):
        case, err, tol = max(vals, key=lambda v: v[1] / max(v[2], 1e-30))
        rows[name] = {"n": len(vals), "worst": err, "tol": tol, "worst_case": case,
                      "all": [[c, e] for c, e, _ in vals]}
        tr.write_line(f"{name:42s} n={len(vals):4d} worst={err:.3e} tol={tol:.0e} ({case})")
    out = ROOT / "gpurun_out"
    if out.is_dir():
        with open(out / "parity_errors.json", "w") as f:
            json.dump(rows, f, indent=1)


def load_golden(name):
    """{case: {field: array}} from tests/golden/<name>.npz (written by make_golden.py)."""
    data = np.load(GOLDEN / f"{name}.npz")
    out = {}
    for key in data.files:
        if "__" in key:
            case, field = key.split("__", 1)
            out.setdefault(case, {})[field] = data[key]
        else:
            out[key] = data[key]
    return out


@pytest.fixture(scope="session")
def golden():
    return load_golden
