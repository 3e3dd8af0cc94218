"""Profiling driver for the benchmark workload (run under ncu on the GPU box).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_mlp.py --steps 2
    ncu --set full --clock-control none --import-source on -k regex:engine \
        -s 4 -c 3 -o gpurun_out/prof python tools/profile_mlp.py --steps 1

Runs the MLP fwd/bwd/upd step (BASELINE config 2) eagerly (no graph, so every
launch is visible to ncu), with the same shapes and kernels as bench.py.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--width", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=2048)
    args = ap.parse_args()
    import torch

    from paper_1906_06440_b200.mlp import MLP

    mlp = MLP(layers=args.layers, width=args.width, batch=args.batch, lr=1e-4, seed=0)
    g = torch.Generator(device="cpu").manual_seed(1)
    nb, cb = args.batch // 64, args.width // 64
    x = (torch.rand(nb, cb, 64, 64, generator=g) * 2 - 1).bfloat16().cuda()
    dy = ((torch.rand(nb, cb, 64, 64, generator=g) * 2 - 1) * 1e-2).bfloat16().cuda()
    mlp.load_input(x, dy)
    for _ in range(args.steps):
        mlp.step()
    torch.cuda.synchronize()
    print(f"ran {args.steps} steps, {mlp.launches_per_step} launches per step")


if __name__ == "__main__":
    main()
