"""GPU parity of the implicit-GEMM conv engine (brk_conv_*: TMA im2col ->
tcgen05 -> TMEM) against the oracle, on bf16 storage with 64-channel blocks.

Integer-valued inputs make the tensor-core sums exact, so the engine must match
the oracle bit for bit after the storage rounding (bf16 for activations, fp32
for dW).  Random inputs are checked at the north-star bf16 tolerance.
"""

import numpy as np
import pytest

import brk_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1906_06440_b200.cnn import (  # noqa: E402
    ConvSpec,
    conv2d_backward_data,
    conv2d_forward,
    conv2d_weight_update,
    engine_plan,
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

# n, c, k, h, w, r, stride — every engine tile kind, partial tiles, pixel walks
# that cross images, the 1x1 stride-2 scatter and non-square maps.
CASES = [
    (2, 64, 64, 8, 8, 3, 1),      # BN=64 single-CTA tiles
    (2, 128, 256, 14, 14, 1, 1),  # CTA pair, BN=256
    (3, 64, 128, 7, 7, 3, 1),     # CTA pair BN=128, N*P*Q=147: partial tile
    (2, 256, 128, 12, 10, 1, 2),  # 1x1 stride 2, rectangular
    (1, 128, 64, 9, 11, 3, 1),    # odd extents
    (4, 64, 256, 5, 5, 1, 1),     # PQ=25: walks cross images; upd tail of 36 zero pixels
    (2, 64, 64, 9, 9, 5, 1),      # 5x5, pad 2
    (2, 512, 128, 7, 7, 3, 1),    # deep C (8 channel blocks)
]


def _tensors(case, rng, integer):
    n, c, k, h, wd, r, st = case
    spec = ConvSpec(n=n, c=c, k=k, h=h, w=wd, r=r, s=r, stride=st)
    if integer:
        i = rng.integers(-1, 2, (n, c, h, wd)).astype(F32)
        w = rng.integers(-1, 2, (k, c, r, r)).astype(F32)
        do = rng.integers(-1, 2, (n, k, spec.out_h, spec.out_w)).astype(F32)
    else:
        i = orc.round_bf16(rng.uniform(-1, 1, (n, c, h, wd)).astype(F32))
        w = orc.round_bf16(rng.uniform(-1, 1, (k, c, r, r)).astype(F32))
        do = orc.round_bf16(rng.uniform(-1, 1, (n, k, spec.out_h, spec.out_w)).astype(F32))
    return spec, i, w, do


def _device_blocked(spec, i, w, do):
    inp, wgt = block_conv_tensors(i, w, 64, 64)
    dob = BlockedTensor(block_conv_input(do, 64).data, 4, {"n": 0, "k": (1, 4), "p": 2, "q": 3})
    return (inp.to("cuda", torch.bfloat16), wgt.to("cuda", torch.bfloat16), dob.to("cuda", torch.bfloat16))


def _run(spec, inp, wgt, dob):
    o = unblock_conv_output(conv2d_forward(spec, inp, wgt, engine=True).to("cpu"))
    di = unblock_conv_input(conv2d_backward_data(spec, dob, wgt, engine=True).to("cpu"))
    dw = unblock_conv_weight(conv2d_weight_update(spec, inp, dob, engine=True).to("cpu"))
    return [np.asarray(t, dtype=np.float64) for t in (o, di, dw)]


def _refs(spec, i, w, do):
    st = spec.stride
    return (orc.conv2d_forward_reference(i, w, st),
            orc.conv2d_backward_data_reference(do, w, (spec.h, spec.w), st),
            orc.conv2d_weight_update_reference(i, do, spec.r, spec.s, st))


@pytest.mark.parametrize("case", CASES)
def test_engine_integer_bit_exact(case):
    spec, i, w, do = _tensors(case, np.random.default_rng(sum(case)), integer=True)
    o, di, dw = _run(spec, *_device_blocked(spec, i, w, do))
    o_ref, di_ref, dw_ref = _refs(spec, i, w, do)
    assert np.array_equal(o, orc.round_bf16(o_ref)), "fwd"
    assert np.array_equal(di, orc.round_bf16(di_ref)), "bwd-data"
    assert np.array_equal(dw, dw_ref), "upd"


@pytest.mark.parametrize("case", CASES[:4])
def test_engine_random_within_bf16_tolerance(case):
    spec, i, w, do = _tensors(case, np.random.default_rng(100 + sum(case)), integer=False)
    got = _run(spec, *_device_blocked(spec, i, w, do))
    for name, g, ref in zip(("fwd", "bwd", "upd"), got, _refs(spec, i, w, do)):
        assert orc.scale_rel_error(g, ref) <= 1e-2, name


@pytest.mark.parametrize("splits", [2, 5])
def test_engine_upd_split_slices_deterministic(monkeypatch, splits):
    case = (4, 128, 128, 14, 14, 3, 1)
    spec, i, w, do = _tensors(case, np.random.default_rng(7), integer=True)
    inp, wgt, dob = _device_blocked(spec, i, w, do)
    monkeypatch.setenv("BRK_CONV_SPLITS", str(splits))
    assert engine_plan(spec, 2)[2] == splits
    dw1 = unblock_conv_weight(conv2d_weight_update(spec, inp, dob, engine=True).to("cpu"))
    dw2 = unblock_conv_weight(conv2d_weight_update(spec, inp, dob, engine=True).to("cpu"))
    ref = orc.conv2d_weight_update_reference(i, do, 3, 3, 1)
    assert np.array_equal(np.asarray(dw1, np.float64), ref)
    assert np.array_equal(np.asarray(dw1), np.asarray(dw2))


def test_engine_matches_grouped_path():
    """The engine and the reference-order grouped BRGEMM path agree (same bf16 inputs)."""
    case = (2, 128, 128, 10, 10, 3, 1)
    spec, i, w, do = _tensors(case, np.random.default_rng(11), integer=False)
    inp, wgt, dob = _device_blocked(spec, i, w, do)
    a = conv2d_forward(spec, inp, wgt, engine=True).data.float()
    b = conv2d_forward(spec, inp, wgt, engine=False).data.float()
    assert (a - b).abs().max().item() <= 1e-2 * b.abs().max().item()


@pytest.mark.parametrize("case", CASES)
def test_engine_tf32_forward(case):
    """fp32 storage, TF32 MMAs on the engine (k-steps of 32 channels: fp32 im2col boxes, the
    weights' MN-major 32-element atoms): integer inputs exact, random inputs within the TF32
    bound of the north star (1e-3), and the same numbers as the grouped TF32 path's bound."""
    rng = np.random.default_rng(300 + sum(case))
    for integer in (True, False):
        spec, i, w, _ = _tensors(case, rng, integer)
        if not integer:
            i = rng.uniform(-1, 1, i.shape).astype(F32)
            w = rng.uniform(-1, 1, w.shape).astype(F32)
        inp, wgt = block_conv_tensors(i, w, 64, 64)
        inp, wgt = inp.to("cuda", torch.float32), wgt.to("cuda", torch.float32)
        got = unblock_conv_output(conv2d_forward(spec, inp, wgt, engine=True, precision="tf32").to("cpu"))
        ref = orc.conv2d_forward_reference(i, w, spec.stride)
        got = np.asarray(got, dtype=np.float64)
        if integer:
            assert np.array_equal(got, ref), case
        else:
            assert orc.scale_rel_error(got, ref) <= 1e-3, case


@pytest.mark.parametrize("case", CASES)
def test_engine_tf32_backward_data(case):
    """fp32 storage, TF32 backward-data on the engine (k-steps of 32 output channels,
    the flipped weights read K-major): integer inputs exact, random inputs within 1e-3."""
    rng = np.random.default_rng(400 + sum(case))
    for integer in (True, False):
        spec, _, w, do = _tensors(case, rng, integer)
        if not integer:
            w = rng.uniform(-1, 1, w.shape).astype(F32)
            do = rng.uniform(-1, 1, do.shape).astype(F32)
        _, wgt = block_conv_tensors(np.zeros((spec.n, spec.c, spec.h, spec.w), F32), w, 64, 64)
        dob = BlockedTensor(block_conv_input(do, 64).data, 4, {"n": 0, "k": (1, 4), "p": 2, "q": 3})
        wgt, dob = wgt.to("cuda", torch.float32), dob.to("cuda", torch.float32)
        got = unblock_conv_input(conv2d_backward_data(spec, dob, wgt, engine=True, precision="tf32").to("cpu"))
        ref = orc.conv2d_backward_data_reference(do, w, (spec.h, spec.w), spec.stride)
        got = np.asarray(got, dtype=np.float64)
        if integer:
            assert np.array_equal(got, ref), case
        else:
            assert orc.scale_rel_error(got, ref) <= 1e-3, case


@pytest.mark.parametrize("case", CASES)
def test_engine_tf32_weight_update(case):
    """fp32 storage, TF32 weight update on the engine (tile-mode blocks of 32 output
    pixels, the taps as coordinate shifts, 32-channel atoms): integer inputs exact, random inputs
    within 1e-3."""
    rng = np.random.default_rng(500 + sum(case))
    for integer in (True, False):
        spec, i, _, do = _tensors(case, rng, integer)
        if not integer:
            i = rng.uniform(-1, 1, i.shape).astype(F32)
            do = rng.uniform(-1, 1, do.shape).astype(F32)
        inp, _ = block_conv_tensors(i, np.zeros((spec.k, spec.c, spec.r, spec.s), F32), 64, 64)
        dob = BlockedTensor(block_conv_input(do, 64).data, 4, {"n": 0, "k": (1, 4), "p": 2, "q": 3})
        inp, dob = inp.to("cuda", torch.float32), dob.to("cuda", torch.float32)
        got = unblock_conv_weight(conv2d_weight_update(spec, inp, dob, engine=True, precision="tf32").to("cpu"))
        ref = orc.conv2d_weight_update_reference(i, do, spec.r, spec.s, spec.stride)
        got = np.asarray(got, dtype=np.float64)
        if integer:
            assert np.array_equal(got, ref), case
        else:
            assert orc.scale_rel_error(got, ref) <= 1e-3, case
