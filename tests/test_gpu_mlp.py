"""GPU parity of the MLP training step (BASELINE config 2) vs the oracle."""

import numpy as np
import pytest

import brk_oracle as orc
from conftest import check_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1906_06440_b200.mlp import MLP  # noqa: E402

B = 64


def blk(a):  # (N, C) -> [N/64][C/64][64][64]
    n, c = a.shape
    return a.reshape(n // B, B, c // B, B).permute(0, 2, 1, 3).contiguous()


def unblk(b):
    nb, cb = b.shape[:2]
    return b.permute(0, 2, 1, 3).reshape(nb * B, cb * B)


def w_dense(wb):  # [Kb][Cb][64c][64k] -> (K, C)
    kb, cb = wb.shape[:2]
    return wb.permute(0, 3, 1, 2).reshape(kb * B, cb * B)


@pytest.mark.parametrize("layers,width,batch", [(2, 256, 256), (4, 512, 384), (4, 1024, 2048), (3, 512, 512)])
def test_mlp_step_matches_oracle(layers, width, batch):
    lr = 0.05
    mlp = MLP(layers=layers, width=width, batch=batch, lr=lr, seed=1)
    g = torch.Generator(device="cpu").manual_seed(2)
    x = (torch.rand(batch, width, generator=g) * 2 - 1).bfloat16()
    dy = (torch.rand(batch, width, generator=g) * 2 - 1).bfloat16()
    ws = [w_dense(w).float().cpu().numpy() for w in mlp.w]
    bs = [b.cpu().numpy().copy() for b in mlp.bias]
    mlp.load_input(blk(x).cuda(), blk(dy).cuda())
    mlp.step()
    torch.cuda.synchronize()
    fwd = orc.mlp_step_reference(ws, bs, x.float().numpy(), dy.float().numpy(), lr=lr, store=orc.round_bf16)
    # forward activations (bf16-stored between layers): 1e-2 scale-relative
    gpu_y = [unblk(mlp.y[l]).float().cpu().numpy() for l in range(1, layers + 1)]
    case = f"{layers}x{width} N={batch}"
    for l in range(1, layers + 1):
        check_parity(f"mlp.y{l}", case, orc.scale_rel_error(gpu_y[l - 1], fwd["y"][l]), 1e-2)
    # backward / update against the oracle fed the GPU's own activations (same ReLU masks)
    ref = orc.mlp_step_reference(ws, bs, x.float().numpy(), dy.float().numpy(), lr=lr, store=orc.round_bf16,
                                 activations=gpu_y)
    for l in range(layers):
        check_parity(f"mlp.dw{l}", case, orc.scale_rel_error(w_dense(mlp.dw[l]).cpu().numpy(), ref["dw"][l]), 1e-2)
        check_parity(f"mlp.db{l}", case, orc.scale_rel_error(mlp.db[l].cpu().numpy(), ref["db"][l]), 1e-2)
        # SGD applied in the upd epilogue (bf16 weights) and in the bias-grad kernel
        w_new = w_dense(mlp.w[l]).float().cpu().numpy()
        # bf16 rounding of the stored weight + lr * (the dW tolerance)
        w_tol = 2.0 ** -8 * np.max(np.abs(ref["w_new"][l])) + lr * 1e-2 * np.max(np.abs(ref["dw"][l]))
        assert np.max(np.abs(w_new - ref["w_new"][l])) <= w_tol, f"w{l}"
        b_tol = lr * 1e-2 * np.max(np.abs(ref["db"][l])) + 1e-6
        assert np.max(np.abs(mlp.bias[l].cpu().numpy() - ref["b_new"][l])) <= b_tol, f"b{l}"
    check_parity("mlp.dx", case, orc.scale_rel_error(unblk(mlp.dz[0]).float().cpu().numpy(), ref["dx"]), 1e-2)


def test_graph_replay_equals_eager_step():
    def make():
        m = MLP(layers=2, width=256, batch=256, lr=0.01, seed=3)
        g = torch.Generator(device="cpu").manual_seed(4)
        x = blk((torch.rand(256, 256, generator=g) * 2 - 1).bfloat16()).cuda()
        dy = blk((torch.rand(256, 256, generator=g) * 2 - 1).bfloat16()).cuda()
        m.load_input(x, dy)
        return m

    eager = make()
    eager.step()
    eager.step()
    graphed = make()
    graphed.capture()          # capture runs one warm-up step eagerly
    graphed.replay()
    torch.cuda.synchronize()
    for l in range(2):
        assert torch.equal(eager.w[l], graphed.w[l])
        assert torch.equal(eager.dw[l], graphed.dw[l])
        assert torch.equal(eager.bias[l], graphed.bias[l])


def test_mlp_step_deterministic():
    outs = []
    for _ in range(2):
        m = MLP(layers=2, width=256, batch=512, lr=0.01, seed=7)
        g = torch.Generator(device="cpu").manual_seed(8)
        m.load_input(blk((torch.rand(512, 256, generator=g) * 2 - 1).bfloat16()).cuda(),
                     blk((torch.rand(512, 256, generator=g) * 2 - 1).bfloat16()).cuda())
        m.step()
        outs.append([t.clone() for t in m.dw + m.db])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_fused_step_matches_per_pass_launches(monkeypatch):
    """brk_mlp_step (one persistent grouped launch) vs the 13 per-pass launches."""
    outs = []
    for fused in ("1", "0"):
        monkeypatch.setenv("BRK_MLP_FUSED", fused)
        mlp = MLP(layers=4, width=512, batch=1024, lr=0.05, seed=3)
        assert mlp.fused == (fused == "1")
        g = torch.Generator(device="cpu").manual_seed(4)
        x = (torch.rand(1024, 512, generator=g) * 2 - 1).bfloat16()
        dy = (torch.rand(1024, 512, generator=g) * 2 - 1).bfloat16()
        mlp.load_input(blk(x).cuda(), blk(dy).cuda())
        for _ in range(2):
            mlp.step()
        torch.cuda.synchronize()
        outs.append([t.float().cpu() for t in mlp.w + mlp.dw + mlp.db + mlp.y[1:]])
    for a, b in zip(*outs):
        assert (a - b).abs().max().item() <= 2e-2 * max(b.abs().max().item(), 1e-6)

