"""MLP step device time with and without an L2 flush between steps (code + data cold vs warm)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_1906_06440_b200.mlp import MLP
mlp = MLP(layers=4, width=1024, batch=2048, lr=1e-4)
mlp.load_input(torch.randn(32, 16, 64, 64, device="cuda").bfloat16(),
               (torch.randn(32, 16, 64, 64, device="cuda") * 1e-2).bfloat16())
mlp.capture()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(200):
    mlp.replay()
for mode in ("flush", "noflush", "flush", "noflush"):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
    torch.cuda.synchronize()
    for i in range(100):
        if mode == "flush":
            flush.fill_(float(i))
        evs[i][0].record()
        mlp.replay()
        evs[i][1].record()
    torch.cuda.synchronize()
    t = sum(a.elapsed_time(b) for a, b in evs) / 100 * 1e3
    print(f"{mode:8s} {t:7.2f} us/step  {51.54e9 / (t * 1e-6) / 1e12:6.1f} TFLOP/s")
