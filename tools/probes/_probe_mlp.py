"""A few fused MLP steps (for ncu captures)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_1906_06440_b200.mlp import MLP
mlp = MLP(layers=4, width=1024, batch=2048, lr=1e-4)
mlp.load_input(torch.randn(32, 16, 64, 64, device="cuda").bfloat16(),
               (torch.randn(32, 16, 64, 64, device="cuda") * 1e-2).bfloat16())
for _ in range(4):
    mlp.step()
torch.cuda.synchronize()
