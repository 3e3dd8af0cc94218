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
    """brk_mlp_step (one persistent launch) vs the 13 per-pass launches over two steps.

    The fused kernel normally sums each tile's k-steps in natural order; the
    per-pass engine rotates the start per tile.  BRK_MLP_FLAGS=1 gives the fused
    kernel the same rotation, so both paths round identically (a different
    summation order flips ReLU masks of activations that round to 0, and at
    lr = 0.05 the second step amplifies that far beyond any tolerance)."""
    outs = []
    monkeypatch.setenv("BRK_MLP_FLAGS", "1")
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



@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("layers,width,batch", [(2, 256, 256), (4, 1024, 2048)])
def test_mlp_tf32_step_matches_oracle(layers, width, batch, fused, monkeypatch):
    """The fp32-storage TF32 step (MlpTF32) at the north-star TF32 tolerance (1e-3): the fused
    persistent launch (brk_mlp_step_dt, BRK_F32) and the per-pass launches."""
    from paper_1906_06440_b200.mlp import MlpTF32

    monkeypatch.setenv("BRK_MLP_FUSED", fused)
    lr = 0.05
    mlp = MlpTF32(layers=layers, width=width, batch=batch, lr=lr, seed=1)
    assert mlp.fused == (fused == "1")
    g = torch.Generator(device="cpu").manual_seed(2)
    x = torch.rand(batch, width, generator=g) * 2 - 1
    dy = torch.rand(batch, width, generator=g) * 2 - 1
    ws = [w_dense(w).cpu().numpy() for w in mlp.w]
    bs = [b.cpu().numpy().copy() for b in mlp.bias]
    mlp.load_input(blk(x).cuda(), blk(dy).cuda())
    mlp.step()
    torch.cuda.synchronize()
    case = f"{layers}x{width} N={batch} {'fused' if fused == '1' else 'per-pass'}"
    fwd = orc.mlp_step_reference(ws, bs, x.numpy(), dy.numpy(), lr=lr)
    gpu_y = [unblk(mlp.y[l]).cpu().numpy() for l in range(1, layers + 1)]
    ins = [x.numpy()] + gpu_y[:-1]
    for l in range(1, layers + 1):
        # each forward pass on identical inputs (the GPU's own previous activation): TF32 1e-3
        ref_l = orc.fc_forward_reference(ws[l - 1], ins[l - 1].T.copy(), "relu", bs[l - 1]).T
        check_parity(f"mlp_tf32.y{l}", case, orc.scale_rel_error(gpu_y[l - 1], ref_l), 1e-3)
        # the whole chain from x compounds one TF32 rounding per layer (recorded, bounded by L x 1e-3)
        check_parity(f"mlp_tf32.chain_y{l}", case, orc.scale_rel_error(gpu_y[l - 1], fwd["y"][l]), l * 1e-3)
    # backward / update, each pass on identical inputs: the GPU's own dz_l and activations
    ys = [x.numpy().astype(np.float64)] + [a.astype(np.float64) for a in gpu_y]
    dz_gpu = [unblk(mlp.dz[l]).cpu().numpy().astype(np.float64) for l in range(layers + 1)]
    check_parity("mlp_tf32.dz_top", case, orc.scale_rel_error(dz_gpu[layers], dy.numpy() * (ys[layers] > 0)), 1e-6)
    for l in range(layers, 0, -1):
        dw_ref = dz_gpu[l].T @ ys[l - 1]
        db_ref = dz_gpu[l].sum(axis=0)
        check_parity(f"mlp_tf32.dw{l - 1}", case, orc.scale_rel_error(w_dense(mlp.dw[l - 1]).cpu().numpy(), dw_ref),
                     1e-3)
        check_parity(f"mlp_tf32.db{l - 1}", case, orc.scale_rel_error(mlp.db[l - 1].cpu().numpy(), db_ref), 1e-3)
        g = dz_gpu[l] @ ws[l - 1].astype(np.float64)
        dz_ref = g * (ys[l - 1] > 0) if l > 1 else g
        check_parity(f"mlp_tf32.dz{l - 1}", case, orc.scale_rel_error(dz_gpu[l - 1], dz_ref), 1e-3)
        # SGD in fp32: W_new = W - lr dW (GPU dW), bias likewise
        w_new = ws[l - 1].astype(np.float64) - lr * w_dense(mlp.dw[l - 1]).cpu().numpy()
        assert np.max(np.abs(w_dense(mlp.w[l - 1]).cpu().numpy() - w_new)) <= 1e-6 * np.max(np.abs(w_new)), f"w{l}"
        b_new = bs[l - 1].astype(np.float64) - lr * mlp.db[l - 1].cpu().numpy()
        assert np.max(np.abs(mlp.bias[l - 1].cpu().numpy() - b_new)) <= 1e-6 * max(np.max(np.abs(b_new)), 1.0), f"b{l}"
    # and the whole backward chain against the oracle from the GPU activations (recorded)
    ref = orc.mlp_step_reference(ws, bs, x.numpy(), dy.numpy(), lr=lr, activations=gpu_y)
    check_parity("mlp_tf32.chain_dx", case, orc.scale_rel_error(unblk(mlp.dz[0]).cpu().numpy(), ref["dx"]),
                 layers * 1e-3)


def test_fused_step_back_to_back_stress():
    """5000 back-to-back graph replays of the headline step (the bench warm-up pattern):
    the cross-CTA dependency protocol (64-column chunk counters, the per-CTA published tile
    ordinal, the exit-ticket counter reset under programmatic dependent launch) must not
    deadlock or fault, and the step stays deterministic."""
    m = MLP(layers=4, width=1024, batch=2048, lr=1e-6, seed=0)
    g = torch.Generator(device="cpu").manual_seed(1)
    m.load_input(blk((torch.rand(2048, 1024, generator=g) * 2 - 1).bfloat16()).cuda(),
                 blk((torch.rand(2048, 1024, generator=g) * 2 - 1).bfloat16()).cuda())
    m.capture()
    for _ in range(5000):
        m.replay()
    torch.cuda.synchronize()
    assert all(torch.isfinite(w.float()).all() for w in m.w)
    assert torch.isfinite(m.grads).all()


def test_fused_step_deterministic_under_back_to_back_replays():
    """The dependency protocol (64-column chunk releases after TMA-store completion, the
    per-CTA published tile ordinal, the counter reset under programmatic dependent launch)
    must hand every consumer complete data: with lr = 0 every step is the same computation,
    so 4000 back-to-back replays must reproduce the first step bit for bit (a stale or
    partial read anywhere in the chain would perturb y, dW, db or dx)."""
    m = MLP(layers=4, width=1024, batch=2048, lr=0.0, seed=0)
    g = torch.Generator(device="cpu").manual_seed(5)
    m.load_input(blk((torch.rand(2048, 1024, generator=g) * 2 - 1).bfloat16()).cuda(),
                 blk((torch.rand(2048, 1024, generator=g) * 2 - 1).bfloat16()).cuda())
    m.capture()
    m.replay()
    torch.cuda.synchronize()
    first = [t.clone() for t in m.dw + m.db + m.y[1:] + m.dz]
    for i in range(40):
        for _ in range(100):
            m.replay()
        torch.cuda.synchronize()
        now = m.dw + m.db + m.y[1:] + m.dz
        for a, b in zip(first, now):
            assert torch.equal(a, b), f"step {100 * (i + 1)}: fused step not reproducible"


def test_fused_tf32_step_deterministic_under_back_to_back_launches():
    """The TF32 variant of the fused step under the same protocol: with lr = 0 every step
    repeats the same computation, so 2000 back-to-back launches must reproduce the first
    step bit for bit."""
    from paper_1906_06440_b200.mlp import MlpTF32

    m = MlpTF32(layers=4, width=1024, batch=2048, lr=0.0, seed=0)
    assert m.fused
    g = torch.Generator(device="cpu").manual_seed(7)
    m.load_input(blk(torch.rand(2048, 1024, generator=g) * 2 - 1).cuda(),
                 blk(torch.rand(2048, 1024, generator=g) * 2 - 1).cuda())
    m.step()
    torch.cuda.synchronize()
    first = [t.clone() for t in m.dw + m.db + m.y[1:] + m.dz]
    for i in range(20):
        for _ in range(100):
            m.step()
        torch.cuda.synchronize()
        for a, b in zip(first, m.dw + m.db + m.y[1:] + m.dz):
            assert torch.equal(a, b), f"step {100 * (i + 1)}: fused TF32 step not reproducible"
