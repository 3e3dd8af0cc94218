"""Shared test fixtures: repo on sys.path, the `gpu` marker, golden-vector loader."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libbrk_sm100.so")


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
