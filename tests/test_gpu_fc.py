"""GPU parity of the FC passes (fwd / bwd-data / weight update / bias) vs the oracle,
on both native paths: the TMA engine (bf16, 64-blocking) and the grouped
batch-list BRGEMM (any blocking, TF32 or BF16)."""

import numpy as np
import pytest

import brk_oracle as orc
from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1906_06440_b200 import _lib, precision  # noqa: E402
from paper_1906_06440_b200.fc import (  # noqa: E402
    Activation,
    FcParams,
    fc_backward_data,
    fc_bias_grad,
    fc_forward,
    fc_weight_update,
)
from paper_1906_06440_b200.tensor import (  # noqa: E402
    BlockedTensor,
    LayoutError,
    block_fc_activation,
    block_weight_2d,
    unblock_fc_activation,
    unblock_weight_2d,
)

TOL = {"tf32": 1e-3, "bf16": 1e-2}
F32 = np.float32


def act_err(got, w, x, act, bias=None):
    """Output error normalised by the GEMM's scale: max|dy| / (max|z| * max g').

    The TF32/BF16 tolerance applies to the batch-reduce result z = W x (+b);
    a Lipschitz activation g maps it to |dy| <= max g' * |dz| (relu 1, sigmoid 1/4).
    """
    z = orc.fc_forward_reference(w, x.T, "identity", bias).T.astype(np.float64)
    y = orc.fc_forward_reference(w, x.T, act, bias).T
    gmax = {"identity": 1.0, "relu": 1.0, "sigmoid": 0.25}[act]
    return float(np.max(np.abs(np.asarray(got, np.float64) - y)) / (np.max(np.abs(z)) * gmax))


def run_fc(w, x, act=Activation.IDENTITY, bias=None, **blk):
    n = x.shape[0]
    p = FcParams.from_dense(w, n, activation=act, bias=bias, **blk)
    return unblock_fc_activation(fc_forward(p, block_fc_activation(x, p.b_n, p.b_c)))


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
@pytest.mark.parametrize("act", ["identity", "relu", "sigmoid"])
def test_golden_fc_forward(prec, act):
    cases = load_golden("fc")
    with precision(prec):
        for ck in (128, 256):
            d = cases[f"ck{ck}_{act}"]
            got = run_fc(d["w"], d["x"], Activation(act))
            assert act_err(got, d["w"], d["x"], act) <= TOL[prec]
            if act == "identity":
                assert orc.scale_rel_error(got, d["oracle"]) <= TOL[prec]


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_integer_kat_bit_exact(prec):
    d = load_golden("fc")["int_relu"]   # N=C=K=128, b=64: bf16 runs the TMA engine
    with precision(prec):
        got = run_fc(d["w"], d["x"], Activation.RELU)
    assert np.array_equal(got, d["y"])


def test_small_blockings_and_identity():
    rng = np.random.default_rng(1)
    x = rng.integers(-4, 5, (8, 16)).astype(F32)
    assert np.array_equal(run_fc(np.eye(16, dtype=F32), x, b_n=4, b_c=8, b_k=8), x)
    w = rng.uniform(-1.0, -0.1, (8, 8)).astype(F32)
    xp = rng.uniform(0.1, 1.0, (4, 8)).astype(F32)
    assert np.array_equal(run_fc(w, xp, Activation.RELU, b_n=2, b_c=4, b_k=4), np.zeros((4, 8), F32))
    w = rng.uniform(-1, 1, (32, 24)).astype(F32)
    x = rng.uniform(-1, 1, (12, 24)).astype(F32)
    for act in Activation:
        got = run_fc(w, x, act, b_n=6, b_c=8, b_k=16)
        assert act_err(got, w, x, act.value) <= 1e-3


def test_layout_errors():
    rng = np.random.default_rng(9)
    w = rng.uniform(-1, 1, (16, 16)).astype(F32)
    p = FcParams.from_dense(w, 8, b_n=4, b_c=8, b_k=8)
    bad = block_fc_activation(rng.uniform(-1, 1, (8, 16)).astype(F32), 2, 8)
    with pytest.raises(LayoutError, match="blocking"):
        fc_forward(p, bad)
    with pytest.raises(ValueError):
        fc_forward(p, block_fc_activation(np.zeros((8, 16), F32), 4, 8), workers=0)


def _device_layer(n, c, k, seed, act=Activation.RELU, b=64, dtype=torch.bfloat16):
    rng = np.random.default_rng(seed)
    w = (rng.uniform(-1, 1, (k, c)) / np.sqrt(c)).astype(F32)
    x = rng.uniform(-1, 1, (n, c)).astype(F32)
    bias = rng.uniform(-0.2, 0.2, k).astype(F32)
    dy = rng.uniform(-1, 1, (n, k)).astype(F32)
    if dtype == torch.bfloat16:  # the oracle sees exactly the bf16 values the GPU sees
        w, x, dy = orc.round_bf16(w), orc.round_bf16(x), orc.round_bf16(dy)
    p = FcParams.from_dense(w, n, b_n=b, b_c=b, b_k=b, activation=act, bias=bias).to("cuda", dtype)
    xb = block_fc_activation(x, b, b).to("cuda", dtype)
    dyb = block_fc_activation(dy, b, b).to("cuda", dtype)
    dyb = BlockedTensor(dyb.data, n_outer=2, logical_dims={"n": (0, 2), "k": (1, 3)})  # output-gradient naming
    return w, x, bias, dy, p, xb, dyb


@pytest.mark.parametrize("shape", [(256, 128, 128), (384, 256, 640), (2048, 1024, 1024)])
def test_engine_fwd_bwd_upd_bias(shape):
    n, c, k = shape
    w, x, bias, dy, p, xb, dyb = _device_layer(n, c, k, seed=n + c)
    before = _lib.launch_count()
    y = fc_forward(p, xb)
    assert _lib.launch_count() - before == 1          # one engine launch for the whole pass
    y_ref = orc.fc_forward_reference(w, x.T, "relu", bias).T
    y_np = unblock_fc_activation(y).float().cpu().numpy()
    assert orc.scale_rel_error(y_np, y_ref) <= TOL["bf16"]
    # bias grad + ReLU mask (dz = dy * (y > 0)) on the GPU's own y
    db, dz = fc_bias_grad(dyb, y)
    y_used = y_np
    dz_ref = dy * (y_used > 0)
    assert np.array_equal(unblock_fc_activation(dz).float().cpu().numpy(), dz_ref)
    assert orc.scale_rel_error(db.cpu().numpy(), dz_ref.astype(np.float64).sum(0)) <= 1e-5
    # bwd-data with the input's ReLU mask fused, and the weight update
    dx = fc_backward_data(p, dz, mask=xb)
    dx_ref = (dz_ref.astype(np.float64) @ w.astype(np.float64)) * (x > 0)
    assert orc.scale_rel_error(unblock_fc_activation(dx).float().cpu().numpy(), dx_ref) <= TOL["bf16"]
    dw = fc_weight_update(p, xb, dz)
    dw_ref = dz_ref.astype(np.float64).T @ x.astype(np.float64)
    assert orc.scale_rel_error(unblock_weight_2d(dw).cpu().numpy(), dw_ref) <= 1e-4  # fp32 out


def test_fused_sgd_update():
    n, c, k = 256, 256, 256
    w, x, bias, dy, p, xb, dyb = _device_layer(n, c, k, seed=5, act=Activation.IDENTITY)
    w_before = unblock_weight_2d(p.w).float().cpu().numpy()
    dw = fc_weight_update(p, xb, dyb, lr=0.01)
    dw_np = unblock_weight_2d(dw).cpu().numpy()
    w_after = unblock_weight_2d(p.w).float().cpu().numpy()
    expect = orc.round_bf16((w_before - 0.01 * dw_np).astype(F32))
    assert np.max(np.abs(w_after - expect)) <= 2 ** -7 * np.max(np.abs(w_before))


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_generic_path_bwd_upd_odd_blocking(prec):
    """Blockings the engine does not serve go through the grouped BRGEMM path."""
    rng = np.random.default_rng(12)
    n, c, k = 24, 40, 48
    w = rng.uniform(-1, 1, (k, c)).astype(F32)
    x = rng.uniform(-1, 1, (n, c)).astype(F32)
    y = orc.fc_forward_reference(w, x.T, "relu").T.copy()
    dy = rng.uniform(-1, 1, (n, k)).astype(F32)
    dx_ref, dw_ref, db_ref = orc.fc_backward_reference(w, x, y, dy, "relu")
    p = FcParams.from_dense(w, n, b_n=8, b_c=8, b_k=16, activation=Activation.RELU)
    with precision(prec):
        db, dz = fc_bias_grad(block_fc_activation(dy, 8, 16), block_fc_activation(y, 8, 16))
        dx = unblock_fc_activation(fc_backward_data(p, dz))
        dw = unblock_weight_2d(fc_weight_update(p, block_fc_activation(x, 8, 8), dz))
    assert orc.scale_rel_error(db, db_ref) <= 1e-5
    assert orc.scale_rel_error(dx, dx_ref) <= TOL[prec]
    assert orc.scale_rel_error(dw, dw_ref) <= TOL[prec]
