"""A/B of the fused MLP step (BASELINE config 2) under environment settings read by
brk_mlp_step at capture time: graph of 10 steps, CUDA events, best of 5 replays.

    python tools/probes/mlp_ab.py BRK_MLP_CHUNK=0 BRK_MLP_CHUNK=1 ...
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch  # noqa: E402

from paper_1906_06440_b200.mlp import MLP, flops_per_step  # noqa: E402


def time_setting(env):
    for k, v in env.items():
        os.environ[k] = v
    m = MLP(layers=4, width=1024, batch=2048, lr=1e-4, seed=0)
    g = torch.Generator(device="cuda").manual_seed(1)
    m.load_input((torch.rand(m.y[0].shape, generator=g, device="cuda") * 2 - 1).bfloat16(),
                 (torch.rand(m.dy.shape, generator=g, device="cuda") * 2 - 1).bfloat16())
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            m.step(s.cuda_stream)
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for _ in range(10):
            m.step(s.cuda_stream)
    best = 1e9
    for _ in range(5):
        with torch.cuda.stream(s):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            graph.replay()
            e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 10 * 1e3)
    for k in env:
        del os.environ[k]
    fl = flops_per_step(4, 2048, 1024, 1024)
    return best, fl / best / 1e6


for arg in sys.argv[1:] or ["BRK_MLP_CHUNK=1"]:
    env = dict(kv.split("=", 1) for kv in arg.split(",") if kv)
    us, tf = time_setting(env)
    print(f"{arg:40s} {us:8.1f} us/step  {tf:7.1f} TFLOP/s  ({tf / 1659.4:.3f} of burst)", flush=True)
