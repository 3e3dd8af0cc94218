"""GPU parity of the BRGEMM family (address / stride / offset / batched) vs the oracle.

Tolerances: integer-valued inputs are bit-exact (exact in
TF32/BF16, exact fp32 accumulation); random inputs scale-relative
max|d|/max|ref| <= 1e-3 (TF32) and <= 1e-2 (BF16).
"""

import numpy as np
import pytest

import brk_oracle as orc
from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1906_06440_b200 import (  # noqa: E402
    BrgemmError,
    BrgemmSpec,
    batched_gemm,
    brgemm,
    brgemm_offset,
    brgemm_strided,
    precision,
)
from paper_1906_06440_b200 import _lib  # noqa: E402

TOL = {"tf32": 1e-3, "bf16": 1e-2}
F32 = np.float32


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_golden_trials(prec):
    cases = load_golden("brgemm")
    with precision(prec):
        for name, d in cases.items():
            if not name.startswith("t"):
                continue
            m, n = d["c0"].shape[1], d["c0"].shape[0]
            k, batch = d["a"].shape[1], d["a"].shape[0]
            spec = BrgemmSpec(m=m, n=n, k=k, batch=batch, beta=float(d["beta"]))
            got = brgemm(list(d["a"]), list(d["b"]), d["c0"].copy(), spec)
            if int(d["integer"]):
                assert np.array_equal(got, d["oracle"]), name
            else:
                assert orc.scale_rel_error(got, d["oracle"]) <= TOL[prec], name


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_acceptance_generator(prec):
    """tests/test_acceptance.py:50-86 generator (seed 2024_08), 250 specs."""
    rng = np.random.default_rng(2024_08)
    with precision(prec):
        for trial in range(250):
            m = int(rng.integers(1, 129))
            n = int(rng.integers(1, 129))
            k = int(rng.integers(1, 513))
            batch = int(rng.integers(0, min(8, 4096 // k) + 1))
            beta = float(rng.integers(0, 2))
            integer = trial % 5 == 0
            draw = (lambda s: rng.integers(-2, 3, size=s).astype(F32)) if integer else \
                (lambda s: rng.uniform(-1, 1, size=s).astype(F32))
            a = [draw((k, m)) for _ in range(batch)]
            b = [draw((n, k)) for _ in range(batch)]
            c0 = draw((n, m))
            spec = BrgemmSpec(m=m, n=n, k=k, batch=batch, beta=beta)
            got = brgemm(a, b, c0.copy(), spec)
            ref = orc.brgemm_reference(a, b, c0, 1.0, beta)
            if integer:
                assert np.array_equal(got, ref), trial
            else:
                assert orc.scale_rel_error(got, ref) <= TOL[prec], trial


def test_config1_stride_brgemm_16x64cubed():
    """BASELINE config 1: stride BRGEMM fp32, batch=16 of 64x64x64."""
    rng = np.random.default_rng([0, 303])
    a = rng.uniform(-1, 1, (16, 64, 64)).astype(F32)
    b = rng.uniform(-1, 1, (16, 64, 64)).astype(F32)
    spec = BrgemmSpec(m=64, n=64, k=64, batch=16, beta=0.0)
    ref = orc.brgemm_reference(list(a), list(b), np.zeros((64, 64), F32), 1.0, 0.0)
    for prec in ("tf32", "bf16"):
        with precision(prec):
            got = brgemm_strided(a, b, 4096, 4096, np.zeros((64, 64), F32), spec)
            assert orc.scale_rel_error(got, ref) <= TOL[prec]
            addr = brgemm(list(a), list(b), np.zeros((64, 64), F32), spec)
            assert np.array_equal(got, addr)  # same kernel, same order: bit-identical


def test_strided_offset_address_equivalence():
    rng = np.random.default_rng(7)
    for m, n, k, batch in [(8, 5, 6, 4), (37, 11, 9, 3), (64, 64, 64, 16), (130, 7, 33, 2)]:
        a = rng.uniform(-1, 1, (batch, k, m)).astype(F32)
        b = rng.uniform(-1, 1, (batch, n, k)).astype(F32)
        spec = BrgemmSpec(m=m, n=n, k=k, batch=batch, beta=0.0)
        addr = brgemm(list(a), list(b), np.zeros((n, m), F32), spec)
        strd = brgemm_strided(a, b, k * m, n * k, np.zeros((n, m), F32), spec)
        offs = brgemm_offset(a, b, [i * k * m for i in range(batch)], [i * n * k for i in range(batch)],
                             np.zeros((n, m), F32), spec)
        assert np.array_equal(addr, strd)
        assert np.array_equal(addr, offs)


@pytest.mark.parametrize("aligned", [True, False])
def test_offset_variant_tf32_views(aligned):
    """TF32 offset variant: entries that are whole rows of the packed buffers (every offset a
    multiple of the block row length) run on the TMA path after the device check; one offset
    inside a row sends the whole launch to the gather path.  Both within the TF32 bound, and
    the TMA launch bit-identical to the stride variant over the same blocks."""
    rng = np.random.default_rng([11, int(aligned)])
    m, n, k, batch, pool = 64, 64, 64, 16, 24
    a_buf = rng.uniform(-1, 1, (pool, k, m)).astype(F32)
    b_buf = rng.uniform(-1, 1, (pool, n, k)).astype(F32)
    pick = rng.integers(0, pool - 1, batch)  # repeats allowed, any order
    a_offs = [int(i) * k * m for i in pick]
    b_offs = [int(i) * n * k for i in pick[::-1]]
    if not aligned:
        a_offs[3] += 8  # inside a row: not one box
    a_blocks = [a_buf.reshape(-1)[o:o + k * m].reshape(k, m) for o in a_offs]
    b_blocks = [b_buf.reshape(-1)[o:o + n * k].reshape(n, k) for o in b_offs]
    spec = BrgemmSpec(m=m, n=n, k=k, batch=batch, beta=1.0)
    c0 = rng.uniform(-1, 1, (n, m)).astype(F32)
    ref = orc.brgemm_reference(a_blocks, b_blocks, c0, 1.0, 1.0)
    with precision("tf32"):
        got = brgemm_offset(a_buf, b_buf, a_offs, b_offs, c0.copy(), spec)
        assert orc.scale_rel_error(got, ref) <= TOL["tf32"]
        if aligned:
            strd = brgemm_strided(np.stack(a_blocks), np.stack(b_blocks), k * m, n * k, c0.copy(), spec)
            assert np.array_equal(got, strd)


def test_edge_cases():
    # empty batch keeps C (tests/test_brgemm.py:45-49)
    c = np.arange(12, dtype=F32).reshape(3, 4)
    assert np.array_equal(brgemm([], [], c.copy(), BrgemmSpec(m=4, n=3, k=2, batch=0, beta=1.0)), c)
    # alpha = beta = 0 clears C (tests/test_brgemm.py:105-112)
    rng = np.random.default_rng(4)
    a = [rng.uniform(-1, 1, (8, 8)).astype(F32) for _ in range(2)]
    b = [rng.uniform(-1, 1, (4, 8)).astype(F32) for _ in range(2)]
    cc = rng.uniform(-1, 1, (4, 8)).astype(F32)
    assert np.array_equal(brgemm(a, b, cc, BrgemmSpec(m=8, n=4, k=8, batch=2, alpha=0.0, beta=0.0)),
                          np.zeros((4, 8), F32))
    # remainder tiles, integer exact (tests/test_brgemm.py:121-129)
    rng = np.random.default_rng(5)
    a = [rng.integers(-2, 3, (9, 37)).astype(F32) for _ in range(2)]
    b = [rng.integers(-2, 3, (11, 9)).astype(F32) for _ in range(2)]
    spec = BrgemmSpec(m=37, n=11, k=9, batch=2, beta=0.0)
    assert np.array_equal(brgemm(a, b, np.zeros((11, 37), F32), spec),
                          orc.brgemm_reference(a, b, np.zeros((11, 37), F32), 1.0, 0.0))
    # zero stride repeats one block, alpha=2 beta=1 (tests/test_brgemm.py:132-140), integer data
    a0 = rng.integers(-2, 3, (3, 4)).astype(F32)
    b0 = rng.integers(-2, 3, (2, 3)).astype(F32)
    c0 = rng.integers(-2, 3, (2, 4)).astype(F32)
    spec = BrgemmSpec(m=4, n=2, k=3, batch=3, alpha=2.0, beta=1.0)
    assert np.array_equal(brgemm_strided(a0, b0, 0, 0, c0.copy(), spec),
                          orc.brgemm_reference([a0] * 3, [b0] * 3, c0, 2.0, 1.0))
    # beta = 0.5 and large extents crossing tiles (m > 256, n > 128)
    a = [rng.integers(-2, 3, (20, 300)).astype(F32) for _ in range(3)]
    b = [rng.integers(-2, 3, (200, 20)).astype(F32) for _ in range(3)]
    c0 = rng.integers(-2, 3, (200, 300)).astype(F32)
    spec = BrgemmSpec(m=300, n=200, k=20, batch=3, beta=0.5)
    assert np.array_equal(brgemm(a, b, c0.copy(), spec), orc.brgemm_reference(a, b, c0, 1.0, 0.5))


def test_overrun_and_contract_errors():
    spec = BrgemmSpec(m=4, n=2, k=3, batch=3)
    with pytest.raises(BrgemmError, match="overruns"):
        brgemm_strided(np.zeros(12, F32), np.zeros(100, F32), 12, 6, np.zeros((2, 4), F32), spec)
    with pytest.raises(BrgemmError, match="batch"):
        brgemm([np.zeros((3, 4), F32)], [], np.zeros((2, 4), F32), spec)


def test_batched_gemm_one_launch():
    rng = np.random.default_rng(11)
    a = [rng.integers(-2, 3, (8, 8)).astype(F32) for _ in range(4)]
    b = [rng.integers(-2, 3, (8, 8)).astype(F32) for _ in range(4)]
    cs = [np.zeros((8, 8), F32) for _ in range(4)]
    before = _lib.launch_count()
    batched_gemm(a, b, cs, BrgemmSpec(m=8, n=8, k=8, batch=4, beta=0.0))
    assert _lib.launch_count() - before == 1
    for ai, bi, ci in zip(a, b, cs):
        assert np.array_equal(ci, orc.brgemm_reference([ai], [bi], np.zeros((8, 8), F32), 1.0, 0.0))


def test_device_tensors_zero_copy_bf16():
    g = torch.Generator(device="cpu").manual_seed(3)
    a = torch.randint(-2, 3, (6, 96, 80), generator=g).float()
    b = torch.randint(-2, 3, (6, 64, 96), generator=g).float()
    ref = orc.brgemm_reference(list(a.numpy()), list(b.numpy()), np.zeros((64, 80), F32), 1.0, 0.0)
    ad, bd = a.cuda().bfloat16(), b.cuda().bfloat16()
    c = torch.zeros(64, 80, device="cuda")
    brgemm(list(ad), list(bd), c, BrgemmSpec(m=80, n=64, k=96, batch=6, beta=0.0))
    assert np.array_equal(c.cpu().numpy(), ref)
    c2 = torch.zeros(64, 80, device="cuda")
    brgemm_strided(ad, bd, 96 * 80, 64 * 96, c2, BrgemmSpec(m=80, n=64, k=96, batch=6, beta=0.0))
    assert torch.equal(c, c2)
