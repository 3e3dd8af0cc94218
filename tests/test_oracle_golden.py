"""Pin the CPU oracle (and the package's host-side logic) to golden vectors
produced by running the reference itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import brk_oracle as orc
from conftest import load_golden

from paper_1906_06440_b200 import plan_tiles
from paper_1906_06440_b200.tensor import (
    block_conv_tensors,
    block_fc_activation,
    block_weight_2d,
    max_rel_error,
    pad_spatial,
    unblock_conv_input,
    unblock_fc_activation,
    unblock_weight_2d,
)


def test_brgemm_oracle_matches_reference_outputs():
    cases = load_golden("brgemm")
    n_int = 0
    for name, d in cases.items():
        if not name.startswith("t"):
            continue
        got = orc.brgemm_reference(list(d["a"]), list(d["b"]), d["c0"], 1.0, float(d["beta"]))
        # the reference oracle and its tiled kernel
        if int(d["integer"]):
            n_int += 1
            assert np.array_equal(got, d["oracle"]), name
            assert np.array_equal(got, d["tiled"]), name
        else:
            assert max_rel_error(got, d["oracle"]) <= 1e-12, name
            assert max_rel_error(got, d["tiled"]) <= 1e-5, name
    assert n_int >= 10


def test_brgemm_stride_and_offset_variants_match_reference():
    d = load_golden("brgemm")
    s = d["strided"]
    a = orc.strided_blocks(s["a"], 48, 6, 8, 4)
    b = orc.strided_blocks(s["b"], 30, 5, 6, 4)
    assert np.array_equal(orc.brgemm_reference(a, b, np.zeros((5, 8), np.float32), 1.0, 0.0), s["got"])
    a2 = orc.offset_blocks(s["a"], [0, 48, 96, 144], 6, 8)
    b2 = orc.offset_blocks(s["b"], [0, 30, 60, 90], 5, 6)
    assert np.array_equal(orc.brgemm_reference(a2, b2, np.zeros((5, 8), np.float32), 1.0, 0.0), s["got"])
    z = d["zero_stride"]
    got = orc.brgemm_reference([z["a"]] * 3, [z["b"]] * 3, z["c0"], 2.0, 1.0)
    assert np.array_equal(got, z["got"])


def test_planner_matches_reference_and_exhaustive_search():
    rows = load_golden("planner")["rows"]
    for m, n, vlen, budget, m_b, n_b, acc, degraded in rows:
        p = plan_tiles(int(m), int(n), vlen=int(vlen), budget=int(budget))
        assert (p.m_b, p.n_b, p.accumulators, int(p.degraded)) == (m_b, n_b, acc, degraded)
        exp = orc.plan_tiles_reference(int(m), int(n), int(vlen), 5, int(budget))
        assert exp[:3] == (m_b, n_b, acc)


@pytest.mark.parametrize("act", ["identity", "relu", "sigmoid"])
def test_fc_oracle_matches_reference(act):
    cases = load_golden("fc")
    for ck in (128, 256):
        d = cases[f"ck{ck}_{act}"]
        got = orc.fc_forward_reference(d["w"], d["x"].T, act).T
        assert max_rel_error(got, d["oracle"]) <= 1e-12
        assert max_rel_error(got, d["y"]) <= 1e-5
        # the blocked restatement (the timed CPU arm) equals the reference's blocked kernel
        wb = block_weight_2d(d["w"], 64, 64).data
        xb = block_fc_activation(d["x"], 64, 64).data
        yb = orc.fc_forward_blocked(wb, xb, act)
        y = yb.transpose(0, 2, 1, 3).reshape(d["y"].shape)
        assert max_rel_error(y, d["y"]) <= 1e-6


def test_fc_integer_and_identity_kats():
    cases = load_golden("fc")
    d = cases["int_relu"]
    assert np.array_equal(orc.fc_forward_reference(d["w"], d["x"].T, "relu").T, d["y"])
    d = cases["identity"]
    assert np.array_equal(d["y"], d["x"])


def test_lstm_oracle_matches_reference():
    cases = load_golden("lstm")
    for name in ("ck64", "ck128", "init_state"):
        d = cases[name]
        w = {g: d[f"w_{g}"] for g in orc.GATES}
        r = {g: d[f"r_{g}"] for g in orc.GATES}
        b = {g: d[f"bias_{g}"] for g in orc.GATES}
        out = orc.lstm_forward_reference(w, r, b, d["x"], d.get("h0"), d.get("s0"))
        assert max_rel_error(out["h"], d["h_oracle"]) <= 1e-12
        assert max_rel_error(out["s"], d["s_oracle"]) <= 1e-12
        if "h" in d:
            assert max_rel_error(out["h"], d["h"]) <= 1e-5
            for g in orc.GATES:
                assert max_rel_error(out["gates"][g], d[f"gate_{g}"]) <= 1e-5


def test_conv_oracle_matches_reference():
    cases = load_golden("conv")
    for name, d in cases.items():
        got = orc.conv2d_forward_reference(d["i"], d["w"], int(d["stride"]))
        if name.startswith("int"):
            assert np.array_equal(got, d["oracle"]), name
        else:
            assert max_rel_error(got, d["oracle"]) <= 1e-9, name
            if "got" in d:
                assert max_rel_error(got, d["got"]) <= 1e-5, name


def test_layouts_match_reference():
    d = load_golden("tensor")
    assert np.array_equal(block_weight_2d(d["w"], 4, 2).data, d["w_blk"])
    assert np.array_equal(unblock_weight_2d(block_weight_2d(d["w"], 4, 2)), d["w"])
    xb = block_fc_activation(d["x"], 3, 4)
    assert np.array_equal(xb.data, d["x_blk"])
    assert np.array_equal(unblock_fc_activation(xb), d["x"])
    bi, bw = block_conv_tensors(d["i"], d["kw"], 3, 2)
    assert np.array_equal(bi.data, d["i_blk"])
    assert np.array_equal(bw.data, d["kw_blk"])
    assert np.array_equal(unblock_conv_input(bi), d["i"])
    assert np.array_equal(pad_spatial(bi, 1, 2).data, d["i_pad"])
    assert max_rel_error(d["x"], d["x"] + np.float32(1e-3)) == pytest.approx(float(d["mre"]), rel=1e-12)


def test_rounding_emulation():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5], np.float32)
    assert np.array_equal(orc.round_bf16(x), np.array([1.0, 1.0, 1.0 + 2 ** -7, -2.5], np.float32))
    t = orc.round_tf32(np.array([1.0 + 2 ** -12, 1.0 + 2 ** -11, 1.0 + 2 ** -10], np.float32))
    assert np.array_equal(t, np.array([1.0, 1.0 + 2 ** -10, 1.0 + 2 ** -10], np.float32))
