"""TF32 on the TMA / tcgen05 engine (kind::tf32): fp32-storage FC passes and the
dense GEMM run on engine_kernel<*, tf32=true, *> with 128 B-swizzled 32-element
atoms (csrc/brk_fc.cu split_layout, csrc/brk_gemm.cu).  North-star tolerance
TF32: scale-relative 1e-3 against the fp64 oracle on the same fp32 inputs;
integer-valued inputs are exact in TF32 and must match bit for bit."""

import numpy as np
import pytest

import brk_oracle as orc
from conftest import check_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1906_06440_b200 import _lib, precision  # noqa: E402
from paper_1906_06440_b200._dense import gemm  # noqa: E402
from paper_1906_06440_b200.fc import (  # noqa: E402
    Activation,
    FcParams,
    fc_backward_data,
    fc_forward,
    fc_weight_update,
)
from paper_1906_06440_b200.tensor import BlockedTensor, block_fc_activation, unblock_fc_activation  # noqa: E402

F32 = np.float32


@pytest.mark.parametrize("m,n,k,a_t,b_t", [(256, 256, 256, False, False), (384, 512, 1000, False, True),
                                           (2048, 1024, 1024, True, False), (1000, 192, 96, True, True)])
def test_dense_gemm_tf32(m, n, k, a_t, b_t):
    rng = np.random.default_rng(m + n + k)
    for integer in (True, False):
        draw = (lambda s: rng.integers(-3, 4, s).astype(F32)) if integer else \
            (lambda s: rng.uniform(-1, 1, s).astype(F32))
        a = draw((k, m) if a_t else (m, k))
        b = draw((k, n) if b_t else (n, k))
        out = torch.empty(m, n, device="cuda")
        n0 = _lib.launch_count()
        gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), out, a_t=a_t, b_t=b_t)
        assert _lib.launch_count() > n0
        am = a.T if a_t else a
        bm = b.T if b_t else b
        ref = am.astype(np.float64) @ bm.astype(np.float64).T
        got = out.cpu().numpy()
        if integer:
            assert np.array_equal(got, ref.astype(F32)), "integer TF32 GEMM not exact"
        else:
            check_parity("tf32.engine.gemm", (m, n, k, a_t, b_t), orc.scale_rel_error(got, ref), 1e-3)


@pytest.mark.parametrize("n,c,k", [(256, 256, 384), (2048, 1024, 1024), (512, 768, 256)])
def test_fc_passes_tf32_engine(n, c, k):
    rng = np.random.default_rng(n + c + k)
    w = rng.uniform(-1, 1, (k, c)).astype(F32) / np.sqrt(c)
    x = rng.uniform(-1, 1, (n, c)).astype(F32)
    bias = rng.uniform(-0.1, 0.1, k).astype(F32)
    dy = rng.uniform(-1, 1, (n, k)).astype(F32)
    params = FcParams.from_dense(w, n, activation=Activation.RELU, bias=bias).to("cuda", torch.float32)
    xb = block_fc_activation(x, 64, 64).to("cuda", torch.float32)
    with precision("tf32"):
        y = fc_forward(params, xb)
    y_h = unblock_fc_activation(y.to("cpu"))
    ref_y = orc.fc_forward_reference(w, x.T, "relu", bias).T
    check_parity("tf32.engine.fc.fwd", (n, c, k), orc.scale_rel_error(y_h, ref_y), 1e-3)
    # backward-data with the fused ReLU mask of the layer input (mask = x > 0)
    dz = BlockedTensor(block_fc_activation(dy, 64, 64).data, 2, {"n": (0, 2), "k": (1, 3)}).to("cuda", torch.float32)
    with precision("tf32"):
        dx = fc_backward_data(params, dz, mask=xb)
        dw = fc_weight_update(params, xb, dz)
    ref_dx = (dy.astype(np.float64) @ w.astype(np.float64)) * (x > 0)
    check_parity("tf32.engine.fc.bwd", (n, c, k), orc.scale_rel_error(unblock_fc_activation(dx.to("cpu")), ref_dx),
                 1e-3)
    dw_dense = dw.to("cpu").to_dense(["k", "c"])
    ref_dw = dy.astype(np.float64).T @ x.astype(np.float64)
    check_parity("tf32.engine.fc.upd", (n, c, k), orc.scale_rel_error(dw_dense, ref_dw), 1e-3)


def test_fc_tf32_integer_bit_exact_and_sgd():
    rng = np.random.default_rng(5)
    n, c, k = 256, 256, 256
    w = rng.integers(-2, 3, (k, c)).astype(F32)
    x = rng.integers(-2, 3, (n, c)).astype(F32)
    dy = rng.integers(-2, 3, (n, k)).astype(F32)
    params = FcParams.from_dense(w, n).to("cuda", torch.float32)
    xb = block_fc_activation(x, 64, 64).to("cuda", torch.float32)
    dz = BlockedTensor(block_fc_activation(dy, 64, 64).data, 2, {"n": (0, 2), "k": (1, 3)}).to("cuda", torch.float32)
    with precision("tf32"):
        y = unblock_fc_activation(fc_forward(params, xb).to("cpu"))
        dx = unblock_fc_activation(fc_backward_data(params, dz).to("cpu"))
        dw = fc_weight_update(params, xb, dz, lr=0.5).to("cpu").to_dense(["k", "c"])
    assert np.array_equal(y, (x.astype(np.float64) @ w.T).astype(F32))
    assert np.array_equal(dx, (dy.astype(np.float64) @ w).astype(F32))
    ref_dw = (dy.astype(np.float64).T @ x).astype(F32)
    assert np.array_equal(dw, ref_dw)
    # fp32 weights: SGD applied after the engine pass (brk_sgd_apply)
    assert np.array_equal(params.w.to("cpu").to_dense(["k", "c"]), (w - 0.5 * ref_dw).astype(F32))
