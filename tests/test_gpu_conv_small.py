"""GPU parity of the small-channel convolution path (C < 64: the ResNet stem) —
explicit im2col + the dense tcgen05 GEMM (brk_conv_im2col / brk_gemm_dense /
brk_conv_col2im) — against the fp64 oracle (reference cnn.py:201-334).

Integer-valued operands keep every sum exact in fp32 (and every bwd-data column
exact in bf16), so results equal the bf16-rounded oracle bit for bit; the grouped
BRGEMM path (engine=False) must agree as well."""

import numpy as np
import pytest

import brk_oracle as orc

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

CASES = [  # (n, c, h, w, r, s, stride, pad)
    (2, 3, 32, 30, 7, 7, 2, 3),   # the ResNet-50 stem geometry, small image
    (3, 3, 17, 17, 3, 3, 1, 1),
    (2, 16, 12, 12, 5, 5, 2, 2),
]


@pytest.mark.parametrize("case", CASES)
def test_small_channel_conv_passes(case):
    n, c, h, w, r, s, st, pad = case
    rng = np.random.default_rng(c * 100 + r)
    spec = ConvSpec(n=n, c=c, k=64, h=h, w=w, r=r, s=s, stride=st, pad_h=pad, pad_w=pad, b_c=c, b_k=64)
    x = rng.integers(-2, 3, (n, c, h, w)).astype(np.float32)
    wt = rng.integers(-1, 2, (64, c, r, s)).astype(np.float32)
    do = rng.integers(-1, 2, (n, 64, spec.out_h, spec.out_w)).astype(np.float32)
    with precision("bf16"):
        inp, wgt = block_conv_tensors(x, wt, c, 64)
        dout = BlockedTensor(block_conv_input(do, 64).data, 4, {"n": 0, "k": (1, 4), "p": 2, "q": 3})
        y = unblock_conv_output(conv2d_forward(spec, inp, wgt))
        dx = unblock_conv_input(conv2d_backward_data(spec, dout, wgt))
        dw = unblock_conv_weight(conv2d_weight_update(spec, inp, dout))
        y_g = unblock_conv_output(conv2d_forward(spec, inp, wgt, engine=False))
        dw_g = unblock_conv_weight(conv2d_weight_update(spec, inp, dout, engine=False))
    ref_y = orc.conv2d_forward_reference(x, wt, stride=st, pad_h=pad, pad_w=pad)
    ref_dx = orc.conv2d_backward_data_reference(do, wt, (h, w), stride=st, pad_h=pad, pad_w=pad)
    ref_dw = orc.conv2d_weight_update_reference(x, do, r, s, stride=st, pad_h=pad, pad_w=pad)
    assert np.array_equal(y, orc.round_bf16(ref_y))
    assert np.array_equal(dx, orc.round_bf16(ref_dx))
    assert np.array_equal(dw, ref_dw)
    assert np.array_equal(y, y_g)
    assert np.array_equal(dw, dw_g)


def test_small_channel_device_tensors_and_launches():
    """Device-resident blocked tensors stay on the device; fwd is im2col + one GEMM launch."""
    from paper_1906_06440_b200 import _lib

    n, c, h, w = 2, 3, 24, 24
    spec = ConvSpec(n=n, c=c, k=64, h=h, w=w, r=7, s=7, stride=2, pad_h=3, pad_w=3, b_c=3, b_k=64)
    g = torch.Generator(device="cpu").manual_seed(1)
    x = torch.randint(-2, 3, (n, c, h, w), generator=g).float().numpy()
    wt = torch.randint(-1, 2, (64, c, 7, 7), generator=g).float().numpy()
    inp, wgt = block_conv_tensors(x, wt, 3, 64)
    inp, wgt = inp.to("cuda"), wgt.to("cuda")
    with precision("bf16"):
        before = _lib.launch_count()
        out = conv2d_forward(spec, inp, wgt)
        torch.cuda.synchronize()
        assert _lib.launch_count() - before == 2
    assert out.on_device
    ref = orc.conv2d_forward_reference(x, wt, stride=2, pad_h=3, pad_w=3)
    assert np.array_equal(unblock_conv_output(out.to("cpu")), orc.round_bf16(ref))
