"""GPU parity of the device layout transforms (brk_layout_transform) with the
host relabelings that are pinned to the reference's own outputs
(tests/test_oracle_golden.py): every block_* / unblock_* / pad_spatial on a
CUDA tensor must produce exactly the bytes the host path produces."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1906_06440_b200 import tensor as T  # noqa: E402
from paper_1906_06440_b200 import _lib  # noqa: E402

F32 = np.float32


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("shape,b", [((2, 64, 56, 56), 64), ((3, 3, 224, 224), 3), ((2, 2048, 7, 7), 64),
                                     ((1, 96, 9, 13), 32)])
def test_conv_input_roundtrip(shape, b):
    x = np.random.default_rng(1).uniform(-1, 1, shape).astype(F32)
    host = T.block_conv_input(x, b)
    dev = T.block_conv_input(_dev(x), b)
    assert np.array_equal(dev.data.cpu().numpy(), host.data)
    assert np.array_equal(T.unblock_conv_input(dev).cpu().numpy(), x)


@pytest.mark.parametrize("shape,bc,bk", [((256, 64, 1, 1), 64, 64), ((64, 3, 7, 7), 3, 64), ((512, 512, 3, 3), 64, 64),
                                         ((48, 40, 3, 3), 8, 16)])
def test_conv_weight_roundtrip(shape, bc, bk):
    w = np.random.default_rng(2).uniform(-1, 1, shape).astype(F32)
    host = T.block_conv_weight(w, bc, bk)
    dev = T.block_conv_weight(_dev(w), bc, bk)
    assert np.array_equal(dev.data.cpu().numpy(), host.data)
    assert np.array_equal(T.unblock_conv_weight(dev).cpu().numpy(), w)


@pytest.mark.parametrize("n,c,bn,bc", [(2048, 1024, 64, 64), (168, 1024, 56, 64), (10, 12, 5, 4)])
def test_fc_layouts(n, c, bn, bc):
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (n, c)).astype(F32)
    assert np.array_equal(T.block_fc_activation(_dev(x), bn, bc).data.cpu().numpy(),
                          T.block_fc_activation(x, bn, bc).data)
    w = rng.uniform(-1, 1, (c, n)).astype(F32)
    if c % bc == 0 and n % bn == 0:
        dev = T.block_weight_2d(_dev(w), bn, bc)
        assert np.array_equal(dev.data.cpu().numpy(), T.block_weight_2d(w, bn, bc).data)
        assert np.array_equal(T.unblock_weight_2d(dev).cpu().numpy(), w)


def test_pad_spatial_and_bf16_conversion():
    x = np.random.default_rng(4).uniform(-1, 1, (2, 128, 14, 14)).astype(F32)
    bt = T.block_conv_input(_dev(x), 64)
    padded = T.pad_spatial(bt, 1, 2)
    assert np.array_equal(padded.data.cpu().numpy(), T.pad_spatial(T.block_conv_input(x, 64), 1, 2).data)
    # fused fp32 -> bf16 conversion equals torch's round-to-nearest-even cast
    view = _dev(x).reshape(2, 2, 64, 14, 14).permute(0, 1, 3, 4, 2)
    got = T.device_copy_view(view, torch.bfloat16)
    assert torch.equal(got, view.contiguous().to(torch.bfloat16))


def test_layout_kernel_bandwidth_sanity():
    """NCHW -> NCHWc of ResNet layer 2's output at N=128 (fp32 -> bf16): a one-pass copy
    must not be slower than 3x the HBM roofline (catches an uncoalesced regression)."""
    x = torch.rand(128, 256, 56, 56, device="cuda")
    view = x.reshape(128, 4, 64, 56, 56).permute(0, 1, 3, 4, 2)
    for _ in range(3):
        T.device_copy_view(view, torch.bfloat16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        T.device_copy_view(view, torch.bfloat16)
    e1.record()
    e1.synchronize()
    sec = e0.elapsed_time(e1) * 1e-3 / 10
    gbs = x.numel() * (4 + 2) / sec / 1e9
    print(f"layout NCHW->NCHWc fp32->bf16: {gbs:.0f} GB/s")
    assert gbs > 6500 / 3, gbs
    assert _lib.launch_count() > 0
