"""Per-tile timeline of the fused MLP step (brk_mlp_step) from in-kernel %globaltimer stamps.
Needs the diagnostics build: make -C paper_1906_06440_b200/csrc diag (selected below via BRK_LIB)."""
import os
import sys
os.environ.setdefault("BRK_LIB", os.path.join(os.path.dirname(__file__), "..", "..", "paper_1906_06440_b200",
                                              "libbrk_sm100_diag.so"))
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1906_06440_b200 import _lib
from paper_1906_06440_b200.mlp import MLP
mlp = MLP(layers=4, width=1024, batch=2048, lr=1e-4)
x = torch.randn(32, 16, 64, 64, device="cuda").bfloat16()
dy = (torch.randn(32, 16, 64, 64, device="cuda") * 1e-2).bfloat16()
mlp.load_input(x, dy)
for _ in range(3):
    mlp.step()
torch.cuda.synchronize()
lib = _lib.load()
ts = torch.zeros(148 * 16 * 8 + 148 * 16, dtype=torch.int64, device="cuda")
lib.brk_diag_set_timestamps(ts.data_ptr())
mlp2 = MLP(layers=4, width=1024, batch=2048, lr=1e-4)  # rebuild params with the diag pointer
mlp2.load_input(x, dy)
mlp2.step()
torch.cuda.synchronize()
lib.brk_diag_set_timestamps(None)
tsn = ts.cpu().numpy().astype(np.int64)
a = tsn[:148 * 128].reshape(148, 16, 8)
uid = tsn[148 * 128:].reshape(148, 16)  # unit of each local tile (lean kernel, diagnostics build)
CS = int(os.environ.get("BRK_MLP_CS", "2"))
a = a[0::CS]  # (first) pair leader CTA of each cluster
uid = uid[0::CS]
valid = a[:, :, 3] > 0
t0 = a[:, :, 0][valid & (a[:, :, 0] > 0)].min()
n_units = 148 // CS
# global order of tiles per pair: u = unit + i * n_units; problems: tile_begin from sizes
import os
lag = int(os.environ.get("BRK_MLP_UPD_LAG", "1"))
names = ["fwd1", "fwd2", "fwd3", "fwd4"]
order = os.environ.get("BRK_MLP_ORDER")
if not order and "BRK_MLP_UPD_LAG" not in os.environ:  # the default chain-first order (brk_fc.cu)
    order = "b4b3b2u4u3u2u1b1"
if order:
    names += [("bwd" if order[i] == "b" else "upd") + order[i + 1] for i in range(0, len(order), 2)]
else:
    for l in range(4, -lag, -1):
        if l >= 1:
            names.append(f"bwd{l}")
        if 1 <= l + lag <= 4:
            names.append(f"upd{l + lag}")
sizes = [(32 if n.startswith("upd") else 64) * 2 // CS for n in names]
begin = np.cumsum([0] + sizes)
rows = []
for unit in range(n_units):
    for i in range(16):
        u = unit + i * n_units if os.environ.get("BRK_MLP_LIST") == "0" else int(uid[unit, i])
        if u >= begin[-1] or not valid[unit, i]:
            continue
        p = np.searchsorted(begin, u, side="right") - 1
        rows.append((p, *(a[unit, i] - t0)))
rows = np.array(rows, dtype=np.float64)
print("prob  tiles  dep_ok(min..max)   mma_start   mma_len(mean)  epi_len(mean)  done(max) | commit->acc acc->stored stored->fenced fenced->released [us] | chunk released (lean kernel)")
for p in range(12):
    r = rows[rows[:, 0] == p]
    print(f"{names[p]:5s} {len(r):4d}  {r[:,1].min()/1e3:7.2f}..{r[:,1].max()/1e3:7.2f}  {r[:,2].mean()/1e3:8.2f}  "
          f"{(r[:,3]-r[:,2]).mean()/1e3:8.2f}  {(r[:,4]-r[:,3]).mean()/1e3:8.2f}  {r[:,4].max()/1e3:8.2f} | "
          f"{(r[:,5]-r[:,3]).mean()/1e3:6.2f} {(r[:,6]-r[:,5]).mean()/1e3:6.2f} {(r[:,7]-r[:,6]).mean()/1e3:6.2f} {(r[:,4]-r[:,7]).mean()/1e3:6.2f}"
          f" | {(r[:,8]-r[:,7]).mean()/1e3:6.2f}")
