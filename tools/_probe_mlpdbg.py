import sys, os
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
from test_gpu_mlp import blk, unblk, w_dense
import brk_oracle as orc
from paper_1906_06440_b200.mlp import MLP
layers, width, batch = 2, 256, 256
lr = 0.05
mlp = MLP(layers=layers, width=width, batch=batch, lr=lr, seed=1)
print("fused", mlp.fused)
g = torch.Generator(device="cpu").manual_seed(2)
x = (torch.rand(batch, width, generator=g) * 2 - 1).bfloat16()
dy = (torch.rand(batch, width, generator=g) * 2 - 1).bfloat16()
ws = [w_dense(w).float().cpu().numpy() for w in mlp.w]
bs = [b.cpu().numpy().copy() for b in mlp.bias]
mlp.load_input(blk(x).cuda(), blk(dy).cuda())
mlp.step(); torch.cuda.synchronize()
gpu_y = [unblk(mlp.y[l]).float().cpu().numpy() for l in range(1, layers + 1)]
ref = orc.mlp_step_reference(ws, bs, x.float().numpy(), dy.float().numpy(), lr=lr, store=orc.round_bf16, activations=gpu_y)
for l in range(layers):
    d = w_dense(mlp.dw[l]).cpu().numpy()
    print(l, "dw err", orc.scale_rel_error(d, ref["dw"][l]), "gpu absmax", np.abs(d).max(), "ref absmax", np.abs(ref["dw"][l]).max(), "nan", np.isnan(d).any())
    print("  db err", orc.scale_rel_error(mlp.db[l].cpu().numpy(), ref["db"][l]))
    print("  dz", orc.scale_rel_error(unblk(mlp.dz[l+1]).float().cpu().numpy(), ref["dz"][l+1]) if "dz" in ref else "")
