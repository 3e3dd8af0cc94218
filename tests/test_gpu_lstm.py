"""GPU parity of the fused LSTM forward and BPTT/weight-update vs the oracle."""

import math

import numpy as np
import pytest

import brk_oracle as orc
from conftest import check_parity, load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1906_06440_b200 import precision  # noqa: E402
from paper_1906_06440_b200.lstm import (  # noqa: E402
    GATE_NAMES,
    LstmCellWeights,
    LstmParams,
    lstm_backward,
    lstm_forward,
)

TOL = {"tf32": 1e-3, "bf16": 1e-2}
F32 = np.float32


def weights_from(d):
    return LstmCellWeights(**{f"w_{g}": d[f"w_{g}"] for g in GATE_NAMES},
                           **{f"r_{g}": d[f"r_{g}"] for g in GATE_NAMES},
                           **{f"bias_{g}": d[f"bias_{g}"] for g in GATE_NAMES})


def oracle_args(wt):
    return ({g: getattr(wt, f"w_{g}") for g in GATE_NAMES}, {g: getattr(wt, f"r_{g}") for g in GATE_NAMES},
            {g: getattr(wt, f"bias_{g}") for g in GATE_NAMES})


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_golden_forward(prec):
    cases = load_golden("lstm")
    for name in ("ck64", "ck128", "init_state"):
        d = cases[name]
        wt = weights_from(d)
        t, n, _ = d["x"].shape
        params = LstmParams.from_dense(wt, t, n)
        with precision(prec):
            seq = lstm_forward(params, d["x"], d.get("h0"), d.get("s0"), keep_gates=True)
        assert orc.scale_rel_error(seq.h, d["h_oracle"]) <= TOL[prec], name
        assert orc.scale_rel_error(seq.s, d["s_oracle"]) <= TOL[prec], name


def test_zero_weight_fixed_point_and_scalar_kat():
    # zero weights: i=f=o=1/2, c=0 -> s_t = s_{t-1}/2, h = 0 exactly (tests/test_lstm.py:79-91)
    wt = LstmCellWeights.zeros(8, 8)
    params = LstmParams.from_dense(wt, 4, 4, b_k=4, b_c=4, b_n=2)
    x = np.random.default_rng(1).uniform(-1, 1, (4, 4, 8)).astype(F32)
    seq = lstm_forward(params, x)
    assert np.array_equal(seq.h, np.zeros_like(seq.h)) and np.array_equal(seq.s, np.zeros_like(seq.s))
    # K=C=1 hand recurrence (tests/test_lstm.py:113-139)
    wt = LstmCellWeights.zeros(1, 1)
    for g in GATE_NAMES:
        getattr(wt, f"w_{g}")[:] = 1.0
        getattr(wt, f"r_{g}")[:] = 1.0
    sig = lambda v: 1.0 / (1.0 + math.exp(-v))  # noqa: E731
    s0 = sig(1.0) * math.tanh(1.0)
    h0 = sig(1.0) * math.tanh(s0)
    pre1 = 1.0 + h0
    s1 = sig(pre1) * s0 + sig(pre1) * math.tanh(pre1)
    h1 = sig(pre1) * math.tanh(s1)
    seq = lstm_forward(LstmParams.from_dense(wt, 2, 1, b_k=1, b_c=1, b_n=1), np.ones((2, 1, 1), F32))
    assert seq.h[0, 0, 0] == pytest.approx(h0, rel=1e-5)  # integer inputs: exact TF32/BF16 products
    assert seq.h[1, 0, 0] == pytest.approx(h1, rel=2e-3)   # h0 enters R as a TF32-rounded value


@pytest.mark.parametrize("shape", [(3, 4, 8, 8, 4), (5, 6, 16, 24, 8), (4, 8, 64, 64, 64), (3, 130, 64, 128, 64)])
@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_forward_backward_vs_oracle(shape, prec):
    t, n, c, k, b = shape
    rng = np.random.default_rng(sum(shape))
    wt = LstmCellWeights.random(rng, c, k)
    x = rng.uniform(-1, 1, (t, n, c)).astype(F32)
    h0 = rng.uniform(-1, 1, (n, k)).astype(F32)
    s0 = rng.uniform(-1, 1, (n, k)).astype(F32)
    dh = rng.uniform(-1, 1, (t, n, k)).astype(F32)
    params = LstmParams.from_dense(wt, t, n, b_k=min(b, k), b_c=min(b, c))
    w, r, bias = oracle_args(wt)
    fwd_ref = orc.lstm_forward_reference(w, r, bias, x, h0, s0)
    with precision(prec):
        seq = lstm_forward(params, x, h0, s0, keep_gates=True)
        grads = lstm_backward(params, x, seq, dh, h0, s0)
    tol = TOL[prec]
    case = f"{shape}"
    check_parity(f"lstm.step.{prec}.h", case, orc.scale_rel_error(seq.h, fwd_ref["h"]), tol)
    check_parity(f"lstm.step.{prec}.s", case, orc.scale_rel_error(seq.s, fwd_ref["s"]), tol)
    # BPTT against the oracle fed the GPU's own forward states (isolates the backward)
    gpu_fwd = {"h": seq.h, "s": seq.s, "gates": seq.gates}
    ref = orc.lstm_backward_reference(w, r, x, gpu_fwd, dh, h0, s0)
    for name in ("dx", "dh0", "ds0"):
        check_parity(f"lstm.step.{prec}.{name}", case, orc.scale_rel_error(getattr(grads, name), ref[name]), tol)
    for g in GATE_NAMES:
        for fld in ("dw", "dr", "db"):
            check_parity(f"lstm.step.{prec}.{fld}", (case, g), orc.scale_rel_error(getattr(grads, fld)[g], ref[fld][g]), tol)


def test_causality_and_determinism():
    rng = np.random.default_rng(7)
    wt = LstmCellWeights.random(rng, 8, 8)
    x = rng.uniform(-1, 1, (6, 4, 8)).astype(F32)
    full = lstm_forward(LstmParams.from_dense(wt, 6, 4, b_k=4, b_c=4, b_n=2), x)
    again = lstm_forward(LstmParams.from_dense(wt, 6, 4, b_k=4, b_c=4, b_n=2), x)
    assert np.array_equal(full.h, again.h)
    for t in (1, 3, 5):
        part = lstm_forward(LstmParams.from_dense(wt, t, 4, b_k=4, b_c=4, b_n=2), x[:t].copy())
        assert np.array_equal(part.h, full.h[:t])


@pytest.mark.parametrize("shape", [(3, 168, 1024, 1024), (6, 200, 128, 256), (2, 40, 64, 64)])
def test_sequence_kernels_vs_oracle(shape):
    """The persistent sequence kernels (brk_lstm_seq_fwd/bwd, bf16) at the
    benchmark width (128 CTAs fwd, 32 four-CTA clusters bwd) and odd sizes."""
    t, n, c, k = shape
    rng = np.random.default_rng(sum(shape))
    wt = LstmCellWeights.random(rng, c, k)
    x = rng.uniform(-1, 1, (t, n, c)).astype(F32)
    h0 = rng.uniform(-1, 1, (n, k)).astype(F32)
    s0 = rng.uniform(-1, 1, (n, k)).astype(F32)
    dh = rng.uniform(-1, 1, (t, n, k)).astype(F32)
    params = LstmParams.from_dense(wt, t, n)
    w, r, bias = oracle_args(wt)
    fwd_ref = orc.lstm_forward_reference(w, r, bias, x, h0, s0)
    with precision("bf16"):
        seq = lstm_forward(params, x, h0, s0, keep_gates=True)
        grads = lstm_backward(params, x, seq, dh, h0, s0)
    case = f"{shape}"
    check_parity("lstm.seq.bf16.h", case, orc.scale_rel_error(seq.h, fwd_ref["h"]), 1e-2)
    check_parity("lstm.seq.bf16.s", case, orc.scale_rel_error(seq.s, fwd_ref["s"]), 1e-2)
    ref = orc.lstm_backward_reference(w, r, x, {"h": seq.h, "s": seq.s, "gates": seq.gates}, dh, h0, s0)
    for name in ("dx", "dh0", "ds0"):
        check_parity(f"lstm.seq.bf16.{name}", case, orc.scale_rel_error(getattr(grads, name), ref[name]), 1e-2)
    for g in GATE_NAMES:
        for fld in ("dw", "dr", "db"):
            check_parity(f"lstm.seq.bf16.{fld}", (case, g), orc.scale_rel_error(getattr(grads, fld)[g], ref[fld][g]), 1e-2)


def test_sequence_and_step_paths_agree(monkeypatch):
    rng = np.random.default_rng(3)
    wt = LstmCellWeights.random(rng, 128, 128)
    x = rng.uniform(-1, 1, (5, 64, 128)).astype(F32)
    with precision("bf16"):
        a = lstm_forward(LstmParams.from_dense(wt, 5, 64), x)
        monkeypatch.setenv("BRK_LSTM_SEQ", "0")
        b = lstm_forward(LstmParams.from_dense(wt, 5, 64), x)
    assert orc.scale_rel_error(a.h, b.h) <= 1e-2


def test_in_place_weight_update_is_seen():
    """device copies of the params are keyed on the source arrays'
    content, so an in-place update (SGD on the blocked weights / biases) is
    used by the next call, as in the reference (which reads params every call)."""
    rng = np.random.default_rng(12)
    wt = LstmCellWeights.random(rng, 64, 64)
    x = rng.uniform(-1, 1, (3, 8, 64)).astype(F32)
    params = LstmParams.from_dense(wt, 3, 8)
    with precision("tf32"):
        lstm_forward(params, x)
        params.w_i.data *= 0.5
        params.bias_f[:] += 0.25
        seq = lstm_forward(params, x)
    w, r, bias = oracle_args(wt)
    w["i"] = w["i"] * 0.5
    bias["f"] = np.asarray(params.bias_f).copy()  # (from_dense shares the bias arrays with wt)
    ref = orc.lstm_forward_reference(w, r, bias, x)
    check_parity("lstm.in_place_update.tf32.h", "3x8x64", orc.scale_rel_error(seq.h, ref["h"]), 1e-3)
