"""GPU parity of the convolution passes (fwd / bwd-data / weight update) vs the oracle."""

import numpy as np
import pytest

import brk_oracle as orc
from conftest import load_golden

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

TOL = {"tf32": 1e-3, "bf16": 1e-2}
F32 = np.float32


def run_fwd(spec, i, w):
    inp, wgt = block_conv_tensors(i, w, spec.b_c, spec.b_k)
    return unblock_conv_output(conv2d_forward(spec, inp, wgt))


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_golden_conv_forward(prec):
    cases = load_golden("conv")
    with precision(prec):
        for name, d in cases.items():
            i, w, st = d["i"], d["w"], int(d["stride"])
            n, c, h, wd = i.shape
            k, _, r, s = w.shape
            kw = dict(b_c=3, b_k=4) if name == "int_stride2" else {}
            spec = ConvSpec(n=n, c=c, k=k, h=h, w=wd, r=r, s=s, stride=st, **kw)
            got = run_fwd(spec, i, w)
            if name.startswith("int"):
                assert np.array_equal(got, d["oracle"]), name
            else:
                assert orc.scale_rel_error(got, d["oracle"]) <= TOL[prec], name


def test_identity_and_integer_kats():
    rng = np.random.default_rng(0)
    i = rng.integers(-3, 4, (2, 8, 5, 5)).astype(F32)
    w = np.eye(8, dtype=F32).reshape(8, 8, 1, 1)
    spec = ConvSpec(n=2, c=8, k=8, h=5, w=5, r=1, s=1, b_c=4, b_k=4)
    assert np.array_equal(run_fwd(spec, i, w), i)
    rng = np.random.default_rng(1)
    spec = ConvSpec(n=1, c=2, k=2, h=4, w=4, r=3, s=3, b_c=2, b_k=2)
    i = rng.integers(-2, 3, (1, 2, 4, 4)).astype(F32)
    w = rng.integers(-2, 3, (2, 2, 3, 3)).astype(F32)
    assert np.array_equal(run_fwd(spec, i, w), orc.conv2d_forward_reference(i, w, 1))


BWD_CASES = [
    # n, c, k, h, w, r, stride, b
    (2, 8, 12, 7, 6, 3, 1, 4),
    (1, 16, 8, 9, 9, 3, 1, 8),
    (2, 6, 4, 8, 8, 1, 2, 2),
    (1, 4, 8, 11, 9, 7, 1, 4),
    (2, 64, 64, 8, 8, 3, 1, 64),
    (2, 128, 64, 14, 14, 1, 2, 64),
]


@pytest.mark.parametrize("case", BWD_CASES)
@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_backward_data_and_update(case, prec):
    n, c, k, h, wd, r, st, b = case
    rng = np.random.default_rng(sum(case))
    spec = ConvSpec(n=n, c=c, k=k, h=h, w=wd, r=r, s=r, stride=st, b_c=min(b, c), b_k=min(b, k))
    i = rng.uniform(-1, 1, (n, c, h, wd)).astype(F32)
    w = rng.uniform(-1, 1, (k, c, r, r)).astype(F32)
    do = rng.uniform(-1, 1, (n, k, spec.out_h, spec.out_w)).astype(F32)
    inp, wgt = block_conv_tensors(i, w, spec.b_c, spec.b_k)
    dob = block_conv_input(do, spec.b_k)
    dob = BlockedTensor(dob.data, n_outer=4, logical_dims={"n": 0, "k": (1, 4), "p": 2, "q": 3})
    with precision(prec):
        di = unblock_conv_input(conv2d_backward_data(spec, dob, wgt))
        dw = unblock_conv_weight(conv2d_weight_update(spec, inp, dob))
    di_ref = orc.conv2d_backward_data_reference(do, w, (h, wd), st)
    dw_ref = orc.conv2d_weight_update_reference(i, do, r, r, st)
    assert orc.scale_rel_error(di, di_ref) <= TOL[prec]
    assert orc.scale_rel_error(dw, dw_ref) <= TOL[prec]


def test_integer_backward_bit_exact():
    rng = np.random.default_rng(5)
    spec = ConvSpec(n=2, c=4, k=4, h=6, w=6, r=3, s=3, b_c=4, b_k=4)
    i = rng.integers(-2, 3, (2, 4, 6, 6)).astype(F32)
    w = rng.integers(-2, 3, (4, 4, 3, 3)).astype(F32)
    do = rng.integers(-2, 3, (2, 4, 6, 6)).astype(F32)
    inp, wgt = block_conv_tensors(i, w, 4, 4)
    dob = BlockedTensor(block_conv_input(do, 4).data, 4, {"n": 0, "k": (1, 4), "p": 2, "q": 3})
    di = unblock_conv_input(conv2d_backward_data(spec, dob, wgt))
    dw = unblock_conv_weight(conv2d_weight_update(spec, inp, dob))
    assert np.array_equal(di, orc.conv2d_backward_data_reference(do, w, (6, 6), 1))
    assert np.array_equal(dw, orc.conv2d_weight_update_reference(i, do, 3, 3, 1))
