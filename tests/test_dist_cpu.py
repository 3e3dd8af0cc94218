"""Data-parallel host logic on CPU (gloo, world_size 2): minibatch sharding,
per-layer gradient all-reduce on the GradientReducer, SGD scaling.

The per-rank gradients are computed by the oracle (there is no GPU here); the
test proves that sharding + sum-all-reduce + lr/world reproduce the
full-batch update, which is exactly what the NCCL path in mlp.py / bench.py
relies on."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import brk_oracle as orc

from paper_1906_06440_b200.dist import GradientReducer, sgd_scale, shard_blocks, shard_range


def test_shard_ranges_cover_exactly():
    for n, world in [(10, 3), (2048, 8), (7, 7), (5, 8)]:
        parts = [shard_range(n, r, world) for r in range(world)]
        assert [i for p in parts for i in p] == list(range(n))
        assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
    rows = [shard_blocks(2048, 64, r, 8) for r in range(8)]
    assert [len(r) for r in rows] == [256] * 8 and rows[-1].stop == 2048
    with pytest.raises(ValueError):
        shard_blocks(100, 64, 0, 2)
    assert sgd_scale(0.1, 4) == pytest.approx(0.025)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        layers, n, c = 3, 64, 16
        ws = [rng.uniform(-1, 1, (c, c)).astype(np.float32) / 4 for _ in range(layers)]
        bs = [rng.uniform(-0.1, 0.1, c).astype(np.float32) for _ in range(layers)]
        x = rng.uniform(-1, 1, (n, c)).astype(np.float32)
        dy = rng.uniform(-1, 1, (n, c)).astype(np.float32)
        rows = shard_blocks(n, 8, rank, world)
        local = orc.mlp_step_reference(ws, bs, x[rows.start:rows.stop], dy[rows.start:rows.stop])
        red = GradientReducer()
        grads = []
        for l in range(layers - 1, -1, -1):  # reverse layer order, as the backward produces them
            g = [torch.from_numpy(local["dw"][l].copy()), torch.from_numpy(local["db"][l].copy())]
            red.submit(g)
            grads.append((l, g))
        red.wait()
        lr = 0.1
        step = sgd_scale(lr, red.world)
        out = {l: (ws[l] - step * g[0].numpy(), bs[l] - step * g[1].numpy()) for l, g in grads}
        full = orc.mlp_step_reference(ws, bs, x, dy, lr=lr / world)  # mean-gradient SGD over the global batch
        err = max(max(np.max(np.abs(out[l][0] - full["w_new"][l])), np.max(np.abs(out[l][1] - full["b_new"][l])))
                  for l in range(layers))
        q.put((rank, float(err)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_allreduce_matches_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err in results:
        assert err <= 1e-5, (rank, err)
