"""GPU acceptance suite on the benchmarked configurations, mirroring the
reference's own acceptance suite (/root/reference/pkg/tests/test_acceptance.py)
and extending it to the north-star passes and precisions.

* ResNet-50: all 20 layer shapes at N=2 with the reference's seeds [11, lid]
  (test_acceptance.py:89-101), in forward, backward-data and weight update, on
  every path a layer can take (implicit-GEMM engine / small-channel stem path
  in bf16, the grouped BRGEMM path in bf16 and TF32), against the fp64 oracle
  on the unrounded fp32 inputs.  Integer-valued inputs: bit-exact.
* The reference's 200 random conv specs (seed 2024_11, rs in {1,3,7}, stride
  in {1,2}; test_acceptance.py:103-125), all three passes, TF32 and bf16.
* LSTM at the benchmark shape T=50, N=168, C=K=1024 forward + BPTT.

Tolerances are the north star's (scale-relative max|got-ref|/max|ref|):
TF32 1e-3, bf16 1e-2.  Every measured error is logged (tests/conftest.py) and
printed in the terminal summary.
"""

import numpy as np
import pytest

import brk_oracle as orc
from conftest import check_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1906_06440_b200 import precision  # noqa: E402
from paper_1906_06440_b200.cnn import (  # noqa: E402
    ConvSpec,
    conv2d_backward_data,
    conv2d_forward,
    conv2d_weight_update,
)
from paper_1906_06440_b200.tensor import (  # noqa: E402
    BlockedTensor,
    block_conv_input,
    block_conv_tensors,
    unblock_conv_input,
    unblock_conv_output,
    unblock_conv_weight,
)

F32 = np.float32
TOL = {"tf32": 1e-3, "bf16": 1e-2}
LAYERS = {row[0]: row for row in orc.RESNET50_ROWS}


def _spec(lid, n=2):
    _, c, k, h, w, r, s, st, _ = LAYERS[lid]
    return ConvSpec(n=n, c=c, k=k, h=h, w=w, r=r, s=s, stride=st)


def _draw(spec, seed, integer=False):
    rng = np.random.default_rng(seed)
    if integer:
        d = lambda shape: rng.integers(-1, 2, shape).astype(F32)  # noqa: E731
    else:
        d = lambda shape: rng.uniform(-1, 1, shape).astype(F32)  # noqa: E731
    i = d((spec.n, spec.c, spec.h, spec.w))
    w = d((spec.k, spec.c, spec.r, spec.s))
    do = d((spec.n, spec.k, spec.out_h, spec.out_w)) if not integer else \
        np.random.default_rng([*np.atleast_1d(seed), 1000]).integers(-1, 2, (spec.n, spec.k, spec.out_h,
                                                                              spec.out_w)).astype(F32)
    return i, w, do


def _do_for(spec, seed):
    """dO from the same generator family with tag +1000 (SURVEY 8d synthetic inputs)."""
    return np.random.default_rng([*np.atleast_1d(seed), 1000]).uniform(
        -1, 1, (spec.n, spec.k, spec.out_h, spec.out_w)).astype(F32)


def _run_passes(spec, i, w, do, prec, engine):
    """fwd / bwd-data / upd through the public API on device tensors of the precision's storage type."""
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    inp, wgt = block_conv_tensors(i, w, spec.b_c, spec.b_k)
    dob = block_conv_input(do, spec.b_k)
    dob = BlockedTensor(dob.data, 4, {"n": 0, "k": (1, 4), "p": 2, "q": 3})
    inp, wgt, dob = inp.to("cuda", dt), wgt.to("cuda", dt), dob.to("cuda", dt)
    with precision(prec):
        o = conv2d_forward(spec, inp, wgt, engine=engine)
        di = conv2d_backward_data(spec, dob, wgt, engine=engine)
        dw = conv2d_weight_update(spec, inp, dob, engine=engine)
    torch.cuda.synchronize()
    return (np.asarray(unblock_conv_output(o.to("cpu")), np.float64),
            np.asarray(unblock_conv_input(di.to("cpu")), np.float64),
            np.asarray(unblock_conv_weight(dw.to("cpu")), np.float64))


def _refs(spec, i, w, do):
    st, ph, pw = spec.stride, spec.pad_h, spec.pad_w
    return (orc.conv2d_forward_reference(i, w, st, ph, pw),
            orc.conv2d_backward_data_reference(do, w, (spec.h, spec.w), st, ph, pw),
            orc.conv2d_weight_update_reference(i, do, spec.r, spec.s, st, ph, pw))


_REF_CACHE: dict = {}


def _layer_case(lid):
    if lid not in _REF_CACHE:
        spec = _spec(lid)
        i, w, _ = _draw(spec, [11, lid])
        do = _do_for(spec, [11, lid])
        _REF_CACHE[lid] = (spec, i, w, do, _refs(spec, i, w, do))
    return _REF_CACHE[lid]


# default path (engine / stem) in bf16, and the grouped BRGEMM path in bf16 and TF32
@pytest.mark.parametrize("path", ["default-bf16", "grouped-bf16", "grouped-tf32"])
@pytest.mark.parametrize("lid", list(range(1, 21)))
def test_resnet_layer_n2_all_passes(lid, path):
    spec, i, w, do, refs = _layer_case(lid)
    kind, prec = path.split("-")
    got = _run_passes(spec, i, w, do, prec, None if kind == "default" else False)
    for name, g, ref in zip(("fwd", "bwd", "upd"), got, refs):
        check_parity(f"resnet.{path}.{name}", f"L{lid}", orc.scale_rel_error(g, ref), TOL[prec])


@pytest.mark.parametrize("lid", list(range(1, 21)))
def test_resnet_layer_n2_integer_bit_exact(lid):
    """Integer-valued inputs ({-1, 0, 1}): every product and partial sum is exact in
    fp32, so the bf16 default path equals the oracle after the storage rounding."""
    spec = _spec(lid)
    i, w, do = _draw(spec, [11, lid], integer=True)
    o, di, dw = _run_passes(spec, i, w, do, "bf16", None)
    o_ref, di_ref, dw_ref = _refs(spec, i, w, do)
    assert np.array_equal(o, orc.round_bf16(o_ref)), "fwd"
    assert np.array_equal(di, orc.round_bf16(di_ref)), "bwd-data"
    assert np.array_equal(dw, dw_ref), "upd"


def _random_specs():
    """The reference's 200 random specs, same generator and draw order (test_acceptance.py:103-125)."""
    rng = np.random.default_rng(2024_11)
    out = []
    for trial in range(200):
        rs = int(rng.choice([1, 3, 7]))
        stride = int(rng.choice([1, 2]))
        h = int(rng.integers(max(2, rs - 2), 17))
        w = int(rng.integers(max(2, rs - 2), 17))
        c = int(rng.integers(1, 65))
        k = int(rng.integers(1, 65))
        n = int(rng.integers(1, 3))
        spec = ConvSpec(n=n, c=c, k=k, h=h, w=w, r=rs, s=rs, stride=stride)
        i_dense = rng.uniform(-1, 1, (n, c, h, w)).astype(F32)
        w_dense = rng.uniform(-1, 1, (k, c, rs, rs)).astype(F32)
        out.append((trial, spec, i_dense, w_dense))
    return out


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_random_conv_specs_all_passes(prec):
    specs = _random_specs()
    assert {s.r for _, s, _, _ in specs} == {1, 3, 7} and any(s.stride == 2 for _, s, _, _ in specs)
    for trial, spec, i, w in specs:
        do = _do_for(spec, [2024_11, trial])
        got = _run_passes(spec, i, w, do, prec, None)
        for name, g, ref in zip(("fwd", "bwd", "upd"), got, _refs(spec, i, w, do)):
            check_parity(f"conv-random200.{prec}.{name}", f"trial{trial}", orc.scale_rel_error(g, ref), TOL[prec])


def test_lstm_benchmark_shape_forward_and_bptt():
    """BASELINE config 3 exactly: T=50, N=168, C=K=1024, bf16 (the benchmarked path)."""
    from paper_1906_06440_b200.lstm import GATE_NAMES, LstmCellWeights, LstmParams, lstm_backward, lstm_forward

    t, n, c, k = 50, 168, 1024, 1024
    rng = np.random.default_rng([22, 1024])
    wt = LstmCellWeights.random(rng, c, k)
    x = rng.uniform(-1, 1, (t, n, c)).astype(F32)
    dh = np.random.default_rng([22, 1024, 1000]).uniform(-1, 1, (t, n, k)).astype(F32)
    params = LstmParams.from_dense(wt, t, n)
    w = {g: getattr(wt, f"w_{g}") for g in GATE_NAMES}
    r = {g: getattr(wt, f"r_{g}") for g in GATE_NAMES}
    b = {g: getattr(wt, f"bias_{g}") for g in GATE_NAMES}
    with precision("bf16"):
        seq = lstm_forward(params, x, keep_gates=True)
        grads = lstm_backward(params, x, seq, dh)
    fwd_ref = orc.lstm_forward_reference(w, r, b, x)
    check_parity("lstm.T50N168.bf16.h", "fwd", orc.scale_rel_error(seq.h, fwd_ref["h"]), 1e-2)
    check_parity("lstm.T50N168.bf16.s", "fwd", orc.scale_rel_error(seq.s, fwd_ref["s"]), 1e-2)
    # BPTT against the oracle fed the GPU's forward states (isolates the backward pass)
    ref = orc.lstm_backward_reference(w, r, x, {"h": seq.h, "s": seq.s, "gates": seq.gates}, dh)
    for name in ("dx", "dh0", "ds0"):
        check_parity(f"lstm.T50N168.bf16.{name}", "bptt", orc.scale_rel_error(getattr(grads, name), ref[name]), 1e-2)
    for g in GATE_NAMES:
        for fld in ("dw", "dr", "db"):
            check_parity(f"lstm.T50N168.bf16.{fld}", g,
                         orc.scale_rel_error(getattr(grads, fld)[g], ref[fld][g]), 1e-2)
    # end to end: BPTT against the oracle's own forward (fp32 inputs throughout)
    ref2 = orc.lstm_backward_reference(w, r, x, fwd_ref, dh)
    for g in GATE_NAMES:
        check_parity("lstm.T50N168.bf16.dw_e2e", g, orc.scale_rel_error(grads.dw[g], ref2["dw"][g]), 1e-2)
    check_parity("lstm.T50N168.bf16.dx_e2e", "bptt", orc.scale_rel_error(grads.dx, ref2["dx"]), 1e-2)


def test_brgemm_accumulate_matches_oracle():
    """brgemm_accumulate (brgemm.py:240-257): acc += sum_i A_i B_i into a float64
    buffer; two calls chain into the same accumulator (the multi-list case)."""
    from paper_1906_06440_b200 import BrgemmSpec, brgemm_accumulate

    rng = np.random.default_rng(31)
    for m, n, k, batch in [(64, 56, 64, 16), (37, 11, 9, 3), (128, 128, 64, 8)]:
        a1 = [rng.integers(-2, 3, (k, m)).astype(F32) for _ in range(batch)]
        b1 = [rng.integers(-2, 3, (n, k)).astype(F32) for _ in range(batch)]
        a2 = [rng.integers(-2, 3, (k, m)).astype(F32) for _ in range(batch)]
        b2 = [rng.integers(-2, 3, (n, k)).astype(F32) for _ in range(batch)]
        acc0 = rng.integers(-5, 6, (n, m)).astype(np.float64)
        acc = acc0.copy()
        spec = BrgemmSpec(m=m, n=n, k=k, batch=batch)
        with precision("tf32"):
            out = brgemm_accumulate(a1, b1, acc, spec)
            assert out is acc
            brgemm_accumulate(a2, b2, acc, spec)
        ref = acc0 + sum(bb.astype(np.float64) @ aa.astype(np.float64) for aa, bb in zip(a1 + a2, b1 + b2))
        assert np.array_equal(acc, ref), (m, n, k, batch)
        # random data within TF32 tolerance
        a = [rng.uniform(-1, 1, (k, m)).astype(F32) for _ in range(batch)]
        b = [rng.uniform(-1, 1, (n, k)).astype(F32) for _ in range(batch)]
        acc = np.zeros((n, m))
        with precision("tf32"):
            brgemm_accumulate(a, b, acc, spec)
        ref = sum(bb.astype(np.float64) @ aa.astype(np.float64) for aa, bb in zip(a, b))
        check_parity("brgemm_accumulate.tf32", (m, n, k, batch), orc.scale_rel_error(acc, ref), 1e-3)
