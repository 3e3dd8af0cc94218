"""GPU parity of the dense row-major GEMM on the engine (brk_gemm_dense): the
batch-reduce over K/64 consecutive slices that the LSTM drivers use for the
input projection, backward-data and weight gradients."""

import numpy as np
import pytest

import brk_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1906_06440_b200._dense import gemm  # noqa: E402


@pytest.mark.parametrize("a_t", [False, True])
@pytest.mark.parametrize("b_t", [False, True])
@pytest.mark.parametrize("shape", [(304, 256, 192), (1024, 512, 8400), (40, 64, 72)])
def test_dense_gemm_integer_exact(shape, a_t, b_t):
    """Integer-valued bf16 operands: exact fp32 sums (any transposition, K tails, split-K)."""
    M, N, K = shape
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    a = torch.randint(-2, 3, (M, K), generator=g).float()
    b = torch.randint(-2, 3, (N, K), generator=g).float()
    ref = a.double() @ b.double().t()
    ad = (a.t() if a_t else a).contiguous().cuda().bfloat16()
    bd = (b.t() if b_t else b).contiguous().cuda().bfloat16()
    out = torch.empty(M, N, device="cuda")
    gemm(ad, bd, out, a_t=a_t, b_t=b_t)
    assert torch.equal(out.cpu().double(), ref)


def test_dense_gemm_bias_relu_bf16_out():
    M, N, K = 520, 384, 640
    g = torch.Generator(device="cpu").manual_seed(9)
    a = (torch.rand(M, K, generator=g) * 2 - 1).bfloat16()
    b = (torch.rand(N, K, generator=g) * 2 - 1).bfloat16()
    bias = torch.rand(N, generator=g) * 2 - 1
    ref = torch.relu(a.double() @ b.double().t() + bias.double())
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    gemm(a.cuda(), b.cuda(), out, bias=bias.cuda(), relu=True)
    assert orc.scale_rel_error(out.float().cpu().numpy(), ref.numpy()) <= 1e-2
