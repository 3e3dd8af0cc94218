"""GPU parity of the small-channel convolution paths (C < 64: the ResNet stem) against
the fp64 oracle (reference cnn.py:201-334): stride-2 convs over <= 4 channels run as
space-to-depth implicit GEMMs (brk_conv_s2d_*), the rest as explicit im2col + the dense
tcgen05 GEMM (brk_conv_im2col / brk_gemm_dense / brk_conv_col2im).

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

CASES = [  # (n, c, h, w, r, s, stride, pad, k)
    (2, 3, 32, 30, 7, 7, 2, 3, 64),   # the ResNet-50 stem geometry, small image (s2d)
    (2, 3, 33, 31, 7, 7, 2, 3, 64),   # odd extents (s2d)
    (2, 4, 20, 22, 5, 5, 2, 2, 128),  # even pad, C = 4, two output blocks (s2d)
    (3, 1, 15, 17, 3, 3, 2, 1, 64),   # C = 1 (s2d)
    (2, 2, 16, 16, 7, 7, 2, 0, 64),   # no padding (s2d)
    (3, 3, 17, 17, 3, 3, 1, 1, 64),   # stride 1: explicit im2col
    (2, 16, 12, 12, 5, 5, 2, 2, 64),  # C = 16: explicit im2col
]


@pytest.mark.parametrize("case", CASES)
def test_small_channel_conv_passes(case):
    n, c, h, w, r, s, st, pad, k = case
    rng = np.random.default_rng(c * 100 + r)
    spec = ConvSpec(n=n, c=c, k=k, h=h, w=w, r=r, s=s, stride=st, pad_h=pad, pad_w=pad, b_c=c, b_k=64)
    x = rng.integers(-2, 3, (n, c, h, w)).astype(np.float32)
    wt = rng.integers(-1, 2, (k, c, r, s)).astype(np.float32)
    do = rng.integers(-1, 2, (n, k, spec.out_h, spec.out_w)).astype(np.float32)
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
        assert _lib.launch_count() - before == 3  # s2d unfold + weight transform + engine conv
    assert out.on_device
    ref = orc.conv2d_forward_reference(x, wt, stride=2, pad_h=3, pad_w=3)
    assert np.array_equal(unblock_conv_output(out.to("cpu")), orc.round_bf16(ref))


def test_s2d_matches_im2col_path_random(monkeypatch):
    """Random bf16 operands at a larger stem-shaped case: the space-to-depth path and the
    explicit-im2col path agree within bf16 output rounding, and both with the oracle."""
    n, c, h, w = 4, 3, 64, 64
    spec = ConvSpec(n=n, c=c, k=64, h=h, w=w, r=7, s=7, stride=2, pad_h=3, pad_w=3, b_c=3, b_k=64)
    rng = np.random.default_rng(7)
    x = orc.round_bf16(rng.uniform(-1, 1, (n, c, h, w)).astype(np.float32))
    wt = orc.round_bf16(rng.uniform(-1, 1, (64, c, 7, 7)).astype(np.float32))
    do = orc.round_bf16(rng.uniform(-1, 1, (n, 64, spec.out_h, spec.out_w)).astype(np.float32))
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("BRK_CONV_S2D", mode)
        with precision("bf16"):
            inp, wgt = block_conv_tensors(x, wt, c, 64)
            dout = BlockedTensor(block_conv_input(do, 64).data, 4, {"n": 0, "k": (1, 4), "p": 2, "q": 3})
            outs[mode] = (unblock_conv_output(conv2d_forward(spec, inp, wgt)),
                          unblock_conv_input(conv2d_backward_data(spec, dout, wgt)),
                          unblock_conv_weight(conv2d_weight_update(spec, inp, dout)))
    ref = (orc.conv2d_forward_reference(x, wt, stride=2, pad_h=3, pad_w=3),
           orc.conv2d_backward_data_reference(do, wt, (h, w), stride=2, pad_h=3, pad_w=3),
           orc.conv2d_weight_update_reference(x, do, 7, 7, stride=2, pad_h=3, pad_w=3))
    for i, name in enumerate(("fwd", "bwd", "upd")):
        for mode in ("1", "0"):
            err = orc.scale_rel_error(outs[mode][i], ref[i])
            assert err <= 1e-2, f"{name} s2d={mode}: {err:.2e}"
