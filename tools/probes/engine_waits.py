"""Where a single-problem engine launch waits (diagnostics build, BRK_LIB -> libbrk_sm100_diag.so):
per-CTA clock64 sums of MMA-waits-for-accumulator, MMA-waits-for-operands, epilogue-waits,
epilogue-busy and producer-waits-for-stage, for one ResNet-50 conv pass.
    python tools/probes/engine_waits.py <layer> <fwd|bwd|upd>"""
import os
import sys
os.environ.setdefault("BRK_LIB", os.path.join(os.path.dirname(__file__), "..", "..", "paper_1906_06440_b200",
                                              "libbrk_sm100_diag.so"))
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1906_06440_b200 import _lib  # noqa: E402
from tools.suites import RESNET50_ROWS  # noqa: E402

lib = _lib.load()
lid, pas = int(sys.argv[1]), sys.argv[2]
_, c, k, h, w, r, s, st, _ = [row for row in RESNET50_ROWS if row[0] == lid][0]
n = 256
pad = (r - 1) // 2
p = (h + 2 * pad - r) // st + 1
geom = (n, c, k, h, w, r, s, st, pad, pad)
x = torch.randn(n, c // 64, h, w, 64, device="cuda").bfloat16()
wt = torch.randn(k // 64, c // 64, r, s, 64, 64, device="cuda").bfloat16()
do = torch.randn(n, k // 64, p, p, 64, device="cuda").bfloat16()
out = torch.empty(n, k // 64, p, p, 64, device="cuda", dtype=torch.bfloat16)
din = torch.empty_like(x)
dw = torch.empty(k // 64, c // 64, r, s, 64, 64, device="cuda")
nb = lib.brk_conv_upd_workspace(*geom)
ws = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
fns = {"fwd": lambda: lib.brk_conv_fwd(x.data_ptr(), wt.data_ptr(), None, out.data_ptr(), *geom, 64, 64, 0, 1, sp),
       "bwd": lambda: lib.brk_conv_bwd_data(do.data_ptr(), wt.data_ptr(), din.data_ptr(), *geom, 64, 64, 1, sp),
       "upd": lambda: lib.brk_conv_upd(x.data_ptr(), do.data_ptr(), dw.data_ptr(), None, 0.0, ws.data_ptr(), nb,
                                       *geom, 64, 64, 1, sp)}
f = fns[pas]
for _ in range(3):
    f()
torch.cuda.synchronize()
G = 148
ts = torch.zeros(G * 16 + G * 8, dtype=torch.int64, device="cuda")
lib.brk_diag_set_timestamps(ts.data_ptr())
f()
torch.cuda.synchronize()
lib.brk_diag_set_timestamps(None)
a = ts.cpu().numpy()
st_ = a[:G * 16].reshape(G, 16)
acc = a[G * 16:].reshape(G, 8)[:, :5] / 1.965e3  # us at 1965 MHz
span = (st_[:, 7] - st_[:, 0]) / 1e3
names = ["mma waits acc", "mma waits operands", "epi waits acc", "epi busy", "producer0 waits stage"]
print(f"L{lid} {pas}: kernel span per CTA {span.mean():.1f} us (max {span.max():.1f})")
lead = acc[0::2]
for i, nm in enumerate(names):
    v = (lead if i < 2 else acc)[:, i]
    print(f"  {nm:22s} mean {v.mean():7.1f} us  max {v.max():7.1f}")
