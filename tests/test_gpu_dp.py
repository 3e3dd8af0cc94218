"""Data parallelism end to end on the GPU: two ranks (gloo, world_size 2) share
cuda:0, each runs the real kernels on its shard of the minibatch, the weight
gradients are all-reduced (sum) and SGD applies lr / world.  The result must
equal the full-batch step computed by the oracle, and both replicas must hold
identical weights afterwards (the initial weights are broadcast from rank 0
even though the ranks are seeded differently).  Covers the three workloads:
MLP (mlp.MLP.step), ResNet-50 convs (train.ResNetConvs), LSTM (train.LstmDP)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather(t):
    """all_gather of a (CUDA) tensor over gloo -> list of host float32 arrays (rank order)."""
    t = t.detach().float().cpu().contiguous()
    out = [torch.empty_like(t) for _ in range(WORLD)]
    dist.all_gather(out, t)
    return [o.numpy() for o in out]


def _mlp(rank, q):
    import brk_oracle as orc
    from paper_1906_06440_b200.mlp import MLP

    B, L, C, n_loc, lr = 64, 2, 256, 256, 0.05
    mlp = MLP(layers=L, width=C, batch=n_loc, lr=lr, seed=rank + 1, process_group=dist.group.WORLD)
    ws0 = [w.clone() for w in mlp.w]
    bs0 = [b.clone() for b in mlp.bias]
    g = torch.Generator(device="cpu").manual_seed(2)
    xg = (torch.rand(WORLD * n_loc, C, generator=g) * 2 - 1).bfloat16()
    dyg = (torch.rand(WORLD * n_loc, C, generator=g) * 2 - 1).bfloat16()
    blk = lambda t: t.reshape(-1, B, C // B, B).permute(0, 2, 1, 3).contiguous()  # noqa: E731
    rows = slice(rank * n_loc, (rank + 1) * n_loc)
    mlp.load_input(blk(xg[rows]).cuda(), blk(dyg[rows]).cuda())
    mlp.step()
    torch.cuda.synchronize()
    wd = lambda t: t.permute(0, 3, 1, 2).reshape(C, C)  # noqa: E731
    same = all(np.array_equal(a, b) for w in mlp.w for a, b in [_gather(w)])
    ws = [wd(w).float().cpu().numpy() for w in ws0]
    bs = [b.cpu().numpy() for b in bs0]
    unblk = lambda t: t.permute(0, 2, 1, 3).reshape(-1, C)  # noqa: E731
    acts = [np.concatenate(_gather(unblk(mlp.y[l]).contiguous())) for l in range(1, L + 1)]
    ref = orc.mlp_step_reference(ws, bs, xg.float().numpy(), dyg.float().numpy(), lr=lr / WORLD,
                                 store=orc.round_bf16, activations=acts)
    err_w = max(float(np.max(np.abs(wd(mlp.w[l]).float().cpu().numpy() - ref["w_new"][l]))
                      / np.max(np.abs(ref["w_new"][l]))) for l in range(L))
    err_dw = max(orc.scale_rel_error(wd(mlp.dw[l]).cpu().numpy(), ref["dw"][l]) for l in range(L))
    err_b = max(float(np.max(np.abs(mlp.bias[l].cpu().numpy() - ref["b_new"][l])))
                / (lr / WORLD * float(np.max(np.abs(ref["db"][l]))) + 1e-12) for l in range(L))
    q.put(("mlp", rank, same, err_w, err_dw, err_b))


def _convs(rank, q):
    import brk_oracle as orc
    from paper_1906_06440_b200.tensor import BlockedTensor, unblock_conv_input, unblock_conv_output, unblock_conv_weight
    from paper_1906_06440_b200.train import ResNetConvs

    net = ResNetConvs(n_global=4, layers=[3, 7, 13], lr=0.01, seed=rank, process_group=dist.group.WORLD, counts=False)
    w0 = [lay.w.clone() for lay in net.layers]
    net.step()
    torch.cuda.synchronize()
    worst, same = 0.0, True
    for lay, w_init in zip(net.layers, w0):
        sp = lay.spec
        x = np.concatenate(_gather(lay.bufs["x"]))
        do = np.concatenate(_gather(lay.bufs["dout"]))
        xd = unblock_conv_input(BlockedTensor(x, 4, {"n": 0, "c": (1, 4), "h": 2, "w": 3}))
        dod = unblock_conv_output(BlockedTensor(do, 4, {"n": 0, "k": (1, 4), "p": 2, "q": 3}))
        dw_full = orc.conv2d_weight_update_reference(xd, dod, sp.r, sp.s, sp.stride, sp.pad_h, sp.pad_w)
        wb = lambda t: BlockedTensor(t, 4, {"k": (0, 5), "c": (1, 4), "r": 2, "s": 3})  # noqa: E731
        dw_got = unblock_conv_weight(wb(lay.dw.cpu().numpy()))
        worst = max(worst, orc.scale_rel_error(dw_got, dw_full))
        w_new = unblock_conv_weight(wb(lay.w.float().cpu().numpy()))
        w_ref = unblock_conv_weight(wb(w_init.float().cpu().numpy())) - 0.01 / WORLD * dw_full
        tol = 2.0 ** -8 * np.max(np.abs(w_ref)) + 0.01 / WORLD * 1e-2 * np.max(np.abs(dw_full))
        same = same and float(np.max(np.abs(w_new - w_ref))) <= tol
        a, b = _gather(lay.w)
        same = same and np.array_equal(a, b)
        # the rank's own forward output is that of its images
        out = unblock_conv_output(BlockedTensor(lay.bufs["out"].float().cpu().numpy(), 4,
                                                {"n": 0, "k": (1, 4), "p": 2, "q": 3}))
        xr = unblock_conv_input(BlockedTensor(lay.bufs["x"].float().cpu().numpy(), 4,
                                              {"n": 0, "c": (1, 4), "h": 2, "w": 3}))
        wd = unblock_conv_weight(wb(w_init.float().cpu().numpy()))
        worst = max(worst, orc.scale_rel_error(out, orc.conv2d_forward_reference(xr, wd, sp.stride)))
    q.put(("conv", rank, same, worst, 0.0, 0.0))


def _lstm(rank, q):
    import brk_oracle as orc
    from paper_1906_06440_b200.train import LstmDP

    net = LstmDP(t_steps=3, n_local=40, c=64, k=128, lr=0.01, seed=0, process_group=dist.group.WORLD,
                 precision="bf16")
    p = net.params
    dense = lambda bt, cols: bt.data.permute(0, 3, 1, 2).reshape(net.K, cols).float().cpu().numpy()  # noqa: E731
    w = {g: dense(getattr(p, f"w_{g}"), net.C) for g in net.gates}
    r = {g: dense(getattr(p, f"r_{g}"), net.K) for g in net.gates}
    b = {g: getattr(p, f"bias_{g}").cpu().numpy().copy() for g in net.gates}
    grads = net.step()
    torch.cuda.synchronize()
    xs, dhs = _gather(net.x), _gather(net.dh)
    tot = {g: 0.0 for g in net.gates}
    for xr, dhr in zip(xs, dhs):
        fwd = orc.lstm_forward_reference(w, r, b, xr)
        ref = orc.lstm_backward_reference(w, r, xr, fwd, dhr)
        for g in net.gates:
            tot[g] = tot[g] + ref["dw"][g].astype(np.float64)
    worst = max(orc.scale_rel_error(grads.dw[g].cpu().numpy(), tot[g]) for g in net.gates)
    same = all(np.array_equal(*_gather(getattr(p, f"w_{g}").data)) for g in net.gates)
    q.put(("lstm", rank, same, worst, 0.0, 0.0))


def _worker(rank, port, which, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "oracle")]
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        {"mlp": _mlp, "conv": _convs, "lstm": _lstm}[which](rank, q)
    except Exception as exc:  # noqa: BLE001 - report to the parent
        q.put((which, rank, False, float("inf"), repr(exc), 0.0))
        raise
    finally:
        dist.destroy_process_group()


def _run(which):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, which, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    return res


def test_mlp_dp_world2_matches_full_batch():
    from conftest import check_parity

    for _, rank, same, err_w, err_dw, err_b in _run("mlp"):
        assert same, f"rank {rank}: replicas differ after the step"
        check_parity("dp.mlp.w_new", rank, err_w, 2.0 ** -7)
        check_parity("dp.mlp.dw", rank, err_dw, 1e-2)
        check_parity("dp.mlp.b_new", rank, err_b, 1e-2)


def test_resnet_convs_dp_world2_matches_full_batch():
    from conftest import check_parity

    for _, rank, same, worst, *_ in _run("conv"):
        assert same, f"rank {rank}: replica weights differ or miss the full-batch SGD step"
        check_parity("dp.conv.dw_fwd", rank, worst, 1e-2)


def test_lstm_dp_world2_matches_full_batch():
    from conftest import check_parity

    for _, rank, same, worst, *_ in _run("lstm"):
        assert same, f"rank {rank}: replicas differ after the step"
        check_parity("dp.lstm.dw", rank, worst, 1e-2)


@pytest.mark.gpu
def test_lstm_dp_sgd_and_refreshed_operands():
    """One rank: the SGD step lands on the public blocked params (views of the dense masters),
    and the operand copies LstmDP refreshes after it equal a rebuild from the params (the
    next forward is bit-identical to one after dropping the caches)."""
    from paper_1906_06440_b200 import precision
    from paper_1906_06440_b200.lstm import lstm_forward
    from paper_1906_06440_b200.train import LstmDP

    torch.cuda.set_device(0)
    net = LstmDP(t_steps=4, n_local=40, c=128, k=128, lr=0.05, seed=3, precision="bf16")
    p = net.params
    dense = lambda bt, cols: bt.data.permute(0, 3, 1, 2).reshape(net.K, cols).clone()  # noqa: E731
    w0 = {g: dense(getattr(p, f"w_{g}"), net.C) for g in net.gates}
    r0 = {g: dense(getattr(p, f"r_{g}"), net.K) for g in net.gates}
    b0 = {g: getattr(p, f"bias_{g}").clone() for g in net.gates}
    grads = net.step()
    torch.cuda.synchronize()
    for g in net.gates:
        close = lambda a, b: torch.allclose(a, b, rtol=1e-6, atol=1e-7)  # noqa: E731 (fp32 a - lr*g, FMA or not)
        assert close(dense(getattr(p, f"w_{g}"), net.C), w0[g] - 0.05 * grads.dw[g])
        assert close(dense(getattr(p, f"r_{g}"), net.K), r0[g] - 0.05 * grads.dr[g])
        assert close(getattr(p, f"bias_{g}"), b0[g] - 0.05 * grads.db[g])
        assert not torch.equal(dense(getattr(p, f"w_{g}"), net.C), w0[g])
    with precision("bf16"):
        h_fast = lstm_forward(p, net.x).h.clone()
        object.__setattr__(p, "_brk_device_cell", None)
        object.__setattr__(p, "_brk_seq_cell", None)
        h_rebuilt = lstm_forward(p, net.x).h
    assert torch.equal(h_fast, h_rebuilt)
