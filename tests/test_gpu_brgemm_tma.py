"""GPU parity of the TMA operand path of the generic BRGEMM (stride / offset variants, bf16).

The stride and offset variants fetch an entry's blocks with one TMA box per
operand when the block does not wrap a row of its buffer's 2-d view; the
address variant always takes the cp.async gather.  With integer-valued inputs
every path is exact, so the TMA results must equal the gather results bit for
bit, and both must equal the fp64 oracle (reference brgemm.py:260-337).
"""

import numpy as np
import pytest

import brk_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1906_06440_b200 import _lib  # noqa: E402

BF16, F32, CBF16 = _lib.BRK_BF16, _lib.BRK_F32, _lib.BRK_COMPUTE_BF16


def ints(g, *shape):
    return torch.randint(-3, 4, shape, generator=g).float()


def run_addr(lib, a_ptrs, b_ptrs, c, jobs, m, n, k, batch, lda, ldb):
    c_ptrs = torch.tensor([c.data_ptr() + j * n * m * 4 for j in range(jobs)], dtype=torch.int64, device="cuda")
    ap = torch.tensor(a_ptrs, dtype=torch.int64, device="cuda")
    bp = torch.tensor(b_ptrs, dtype=torch.int64, device="cuda")
    _lib.check(lib.brk_brgemm_addr(ap.data_ptr(), bp.data_ptr(), c_ptrs.data_ptr(), jobs, m, n, k, batch, lda, ldb,
                                   m, 1.0, 0.0, BF16, F32, CBF16, None))
    torch.cuda.synchronize()


@pytest.mark.parametrize("m,n,k,batch,jobs", [(64, 64, 64, 16, 300), (128, 256, 128, 3, 40), (64, 100, 192, 5, 37),
                                              (256, 128, 64, 4, 20), (192, 64, 64, 2, 9)])
def test_stride_tma_matches_gather_and_oracle(m, n, k, batch, jobs):
    lib = _lib.load()
    g = torch.Generator(device="cpu").manual_seed(m + n + k)
    a = ints(g, jobs, batch, k, m).cuda().bfloat16()
    b = ints(g, jobs, batch, n, k).cuda().bfloat16()
    c = torch.zeros(jobs, n, m, device="cuda")
    _lib.check(lib.brk_brgemm_stride(a.data_ptr(), b.data_ptr(), k * m, n * k, c.data_ptr(), jobs, batch * k * m,
                                     batch * n * k, n * m, m, n, k, batch, m, k, m, 1.0, 0.0, BF16, F32, CBF16, None))
    torch.cuda.synchronize()
    c2 = torch.zeros_like(c)
    run_addr(lib, [a[j, i].data_ptr() for j in range(jobs) for i in range(batch)],
             [b[j, i].data_ptr() for j in range(jobs) for i in range(batch)], c2, jobs, m, n, k, batch, m, k)
    assert torch.equal(c, c2)
    for j in (0, jobs // 2, jobs - 1):
        ref = orc.brgemm_reference(list(a[j].float().cpu().numpy()), list(b[j].float().cpu().numpy()),
                                   np.zeros((n, m), np.float32), 1.0, 0.0)
        assert np.array_equal(c[j].cpu().numpy(), ref)


def test_offset_tma_with_wrapping_blocks():
    """Blocks carved out of wider matrices at arbitrary (8-aligned) offsets: entries whose
    block wraps a row of the 2-d view take the gather, the rest TMA — same bits as the
    address variant."""
    lib = _lib.load()
    m, n, k, batch, jobs = 64, 64, 128, 6, 24
    lda, ldb = 3 * m + 8, 2 * k + 24  # row strides of the buffers the blocks live in
    g = torch.Generator(device="cpu").manual_seed(11)
    rows_a, rows_b = 4 * k, 4 * n
    a = ints(g, rows_a * lda).cuda().bfloat16()
    b = ints(g, rows_b * ldb).cuda().bfloat16()
    rng = np.random.default_rng(5)
    a_off = []
    b_off = []
    for _ in range(jobs * batch):
        ra, ca = rng.integers(0, rows_a - k), int(rng.integers(0, (lda - 8) // 8)) * 8  # some wrap: ca + m > lda
        rb, cb = rng.integers(0, rows_b - n), int(rng.integers(0, (ldb - 8) // 8)) * 8
        a_off.append(min(int(ra * lda + ca), a.numel() - (k - 1) * lda - m))
        b_off.append(min(int(rb * ldb + cb), b.numel() - (n - 1) * ldb - k))
    wraps = sum((o % lda) + m > lda for o in a_off) + sum((o % ldb) + k > ldb for o in b_off)
    assert 0 < wraps < 2 * jobs * batch
    c = torch.zeros(jobs, n, m, device="cuda")
    c_ptrs = torch.tensor([c[j].data_ptr() for j in range(jobs)], dtype=torch.int64, device="cuda")
    ao = torch.tensor(a_off, dtype=torch.int64, device="cuda")
    bo = torch.tensor(b_off, dtype=torch.int64, device="cuda")
    _lib.check(lib.brk_brgemm_offs(a.data_ptr(), b.data_ptr(), ao.data_ptr(), bo.data_ptr(), c_ptrs.data_ptr(), jobs,
                                   m, n, k, batch, lda, ldb, m, 1.0, 0.0, BF16, F32, CBF16, None))
    torch.cuda.synchronize()
    c2 = torch.zeros_like(c)
    run_addr(lib, [a.data_ptr() + 2 * o for o in a_off], [b.data_ptr() + 2 * o for o in b_off], c2, jobs, m, n, k,
             batch, lda, ldb)
    assert torch.equal(c, c2)
    a_np, b_np = a.float().cpu().numpy(), b.float().cpu().numpy()
    for j in (0, jobs - 1):
        ab = [np.lib.stride_tricks.as_strided(a_np[a_off[j * batch + i]:], (k, m), (lda * 4, 4)) for i in range(batch)]
        bb = [np.lib.stride_tricks.as_strided(b_np[b_off[j * batch + i]:], (n, k), (ldb * 4, 4)) for i in range(batch)]
        ref = orc.brgemm_reference(ab, bb, np.zeros((n, m), np.float32), 1.0, 0.0)
        assert np.array_equal(c[j].cpu().numpy(), ref)


def test_python_address_api_routes_one_storage_lists_to_offsets():
    """brgemm() with block lists from one allocation runs as the offset variant (TMA for
    aligned blocks); lists spanning allocations keep the address variant — same bits."""
    from paper_1906_06440_b200 import BrgemmSpec, brgemm, brgemm_strided

    g = torch.Generator(device="cpu").manual_seed(21)
    m, n, k, batch = 128, 64, 128, 8
    a = ints(g, batch, k, m).cuda().bfloat16()
    b = ints(g, batch, n, k).cuda().bfloat16()
    spec = BrgemmSpec(m=m, n=n, k=k, batch=batch, beta=0.0)
    c1 = torch.zeros(n, m, device="cuda")
    brgemm(list(a), list(b), c1, spec)  # one storage per operand -> offsets (reversed order below too)
    c2 = torch.zeros(n, m, device="cuda")
    brgemm_strided(a, b, k * m, n * k, c2, spec)
    assert torch.equal(c1, c2)
    c3 = torch.zeros(n, m, device="cuda")
    brgemm([x.clone() for x in a], [y.clone() for y in b], c3, spec)  # separate allocations -> addresses
    assert torch.equal(c1, c3)
    ref = orc.brgemm_reference(list(a.float().cpu().numpy()), list(b.float().cpu().numpy()),
                               np.zeros((n, m), np.float32), 1.0, 0.0)
    assert np.array_equal(c1.cpu().numpy(), ref)
    c4 = torch.zeros(n, m, device="cuda")
    brgemm(list(a)[::-1], list(b)[::-1], c4, spec)  # offsets need not be ordered
    ref4 = orc.brgemm_reference(list(a.float().cpu().numpy())[::-1], list(b.float().cpu().numpy())[::-1],
                                np.zeros((n, m), np.float32), 1.0, 0.0)
    assert np.array_equal(c4.cpu().numpy(), ref4)


def test_brgemm_beats_split_gemm():
    """Reference tests/test_acceptance.py:268-292: the batch-reduce GEMM (reduction kept in
    TMEM) beats the split-GEMM formulation (one launch per batch entry, C accumulated through
    memory) by >= 1.2x at the config-1 shape; both compute the same sums."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    from suites import split_gemm_baseline

    r = split_gemm_baseline(iters=5)
    assert r["max_rel_diff"] <= 1e-5
    assert r["speedup"] >= 1.2, r


@pytest.mark.parametrize("m,n,k,batch,jobs", [(64, 64, 64, 16, 300), (128, 100, 128, 3, 40), (256, 128, 64, 4, 20)])
def test_addr_views_match_gather(m, n, k, batch, jobs):
    """brk_brgemm_addr_views: entries inside the registered views take TMA, the rest (a second
    allocation, a block that would run past its view) the gather; bit-identical to the plain
    address variant and exact against the oracle on integer inputs."""
    lib = _lib.load()
    g = torch.Generator(device="cpu").manual_seed(m * 3 + jobs)
    a = ints(g, jobs, batch, k, m).cuda().bfloat16()
    b = ints(g, jobs, batch, n, k).cuda().bfloat16()
    other_a = ints(g, batch, k, m).cuda().bfloat16()  # outside the A view
    a_ptrs = [a[j, i].data_ptr() for j in range(jobs) for i in range(batch)]
    b_ptrs = [b[j, i].data_ptr() for j in range(jobs) for i in range(batch)]
    for i in range(batch):  # job 1 reads its A blocks from another allocation
        a_ptrs[1 * batch + i] = other_a[i].data_ptr()
    c = torch.zeros(jobs, n, m, device="cuda")
    c_ptrs = torch.tensor([c.data_ptr() + j * n * m * 4 for j in range(jobs)], dtype=torch.int64, device="cuda")
    ap = torch.tensor(a_ptrs, dtype=torch.int64, device="cuda")
    bp = torch.tensor(b_ptrs, dtype=torch.int64, device="cuda")
    # the B view ends one block early: the last job's last block would run past it -> gather
    _lib.check(lib.brk_brgemm_addr_views(ap.data_ptr(), bp.data_ptr(), c_ptrs.data_ptr(), a.data_ptr(), a.numel(),
                                         b.data_ptr(), b.numel() - n * k // 2, jobs, m, n, k, batch, m, k, m, 1.0,
                                         0.0, BF16, F32, CBF16, None))
    torch.cuda.synchronize()
    c2 = torch.zeros_like(c)
    run_addr(lib, a_ptrs, b_ptrs, c2, jobs, m, n, k, batch, m, k)
    assert torch.equal(c, c2)
    for j in (0, 1, jobs - 1):
        aj = other_a if j == 1 else a[j]
        ref = orc.brgemm_reference(list(aj.float().cpu().numpy()), list(b[j].float().cpu().numpy()),
                                   np.zeros((n, m), np.float32), 1.0, 0.0)
        assert np.array_equal(c[j].cpu().numpy(), ref)


@pytest.mark.parametrize("m,n,k,batch,jobs", [(32, 32, 32, 16, 1184), (16, 24, 8, 7, 300), (64, 32, 32, 5, 400),
                                              (40, 20, 24, 9, 150), (32, 128, 32, 3, 200), (32, 32, 32, 1, 999),
                                              (8, 8, 16, 64, 333)])
def test_small_blocks_warp_stages_and_compact_ring(m, n, k, batch, jobs):
    """Small blocks: m = k = 32 take 64B-swizzle TMA boxes (stride, offset), other small
    shapes and the address variant the gather path with one warp per stage (and, for
    k <= 32 and one 64-column B atom, the compact 16-stage ring); both compact layouts let
    the M = 128 MMAs read rows of the next stages.  Stride, offset and address variants
    bit-identical and equal to the fp64 oracle on integer inputs, every job checked (a
    stage read from a wrong slot would show)."""
    lib = _lib.load()
    g = torch.Generator(device="cpu").manual_seed(7 * m + n + k + batch)
    a = ints(g, jobs, batch, k, m).cuda().bfloat16()
    b = ints(g, jobs, batch, n, k).cuda().bfloat16()
    c = torch.full((jobs, n, m), float("nan"), device="cuda")
    _lib.check(lib.brk_brgemm_stride(a.data_ptr(), b.data_ptr(), k * m, n * k, c.data_ptr(), jobs, batch * k * m,
                                     batch * n * k, n * m, m, n, k, batch, m, k, m, 1.0, 0.0, BF16, F32, CBF16, None))
    torch.cuda.synchronize()
    c2 = torch.zeros_like(c)
    run_addr(lib, [a[j, i].data_ptr() for j in range(jobs) for i in range(batch)],
             [b[j, i].data_ptr() for j in range(jobs) for i in range(batch)], c2, jobs, m, n, k, batch, m, k)
    assert torch.equal(c, c2)
    # offset variant (m = k = 32: 64B-swizzle boxes after the device box check)
    ji = torch.arange(jobs, device="cuda")[:, None] * batch + torch.arange(batch, device="cuda")[None, :]
    a_off = (ji * (k * m)).reshape(-1).contiguous()
    b_off = (ji * (n * k)).reshape(-1).contiguous()
    c_ptr = (c.data_ptr() + torch.arange(jobs, device="cuda") * (n * m * 4)).contiguous()
    c3 = c.clone()
    c.fill_(float("nan"))
    _lib.check(lib.brk_brgemm_offs(a.data_ptr(), b.data_ptr(), a_off.data_ptr(), b_off.data_ptr(), c_ptr.data_ptr(),
                                   jobs, m, n, k, batch, m, k, m, 1.0, 0.0, BF16, F32, CBF16, None))
    torch.cuda.synchronize()
    assert torch.equal(c, c3)
    ref = torch.einsum("jikm,jink->jnm", a.double(), b.double())  # exact for these integer inputs
    assert torch.equal(c.double(), ref)
    ref0 = orc.brgemm_reference(list(a[0].float().cpu().numpy()), list(b[0].float().cpu().numpy()),
                                np.zeros((n, m), np.float32), 1.0, 0.0)
    assert np.array_equal(c[0].cpu().numpy(), ref0)


@pytest.mark.parametrize("m,n,k,batch,jobs", [(16, 16, 32, 9, 300), (8, 16, 8, 5, 200), (32, 8, 64, 3, 150),
                                              (16, 128, 16, 4, 100)])
def test_small_blocks_tf32_gather(m, n, k, batch, jobs):
    """fp32 blocks with TF32 MMAs on the gather path (converting loads; one warp per stage when
    a stage is <= 4 copies per lane): exact on small-integer inputs, every job checked."""
    lib = _lib.load()
    g = torch.Generator(device="cpu").manual_seed(11 * m + n + k)
    a = ints(g, jobs, batch, k, m).cuda()
    b = ints(g, jobs, batch, n, k).cuda()
    c = torch.full((jobs, n, m), float("nan"), device="cuda")
    _lib.check(lib.brk_brgemm_stride(a.data_ptr(), b.data_ptr(), k * m, n * k, c.data_ptr(), jobs, batch * k * m,
                                     batch * n * k, n * m, m, n, k, batch, m, k, m, 1.0, 0.0, F32, F32,
                                     _lib.BRK_COMPUTE_TF32, None))
    torch.cuda.synchronize()
    ref = torch.einsum("jikm,jink->jnm", a.double(), b.double())
    assert torch.equal(c.double(), ref)
