"""Stamped timeline of CTA 0 in one m=n=k=32, batch 16 stride BRGEMM launch (diagnostics build:
BRK_LIB=paper_1906_06440_b200/libbrk_sm100_diag.so)."""
import ctypes
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch  # noqa: E402

from paper_1906_06440_b200 import _lib  # noqa: E402

lib = _lib.load()
m = n = k = int(os.environ.get("M", "32"))
batch, jobs = int(os.environ.get("B", "16")), 1184
a = torch.randn(jobs * batch * k * m, device="cuda").bfloat16()
b = torch.randn(jobs * batch * n * k, device="cuda").bfloat16()
c = torch.empty(jobs * n * m, device="cuda")
ts = torch.zeros(512, dtype=torch.int64, device="cuda")
lib.brk_diag_set_timestamps.argtypes = [ctypes.c_void_p]


def run():
    _lib.check(lib.brk_brgemm_stride(a.data_ptr(), b.data_ptr(), k * m, n * k, c.data_ptr(), jobs, batch * k * m,
                                     batch * n * k, n * m, m, n, k, batch, m, k, m, 1.0, 0.0, _lib.BRK_BF16,
                                     _lib.BRK_F32, _lib.BRK_COMPUTE_BF16, 0))


for _ in range(3):
    run()
torch.cuda.synchronize()
lib.brk_diag_set_timestamps(ts.data_ptr())
run()
torch.cuda.synchronize()
lib.brk_diag_set_timestamps(None)
t = ts.cpu().tolist()
t0 = min(x for x in t if x > 0)
us = lambda x: (x - t0) / 1e3 if x > 0 else float("nan")  # noqa: E731
print("stage  issue   full   mma")
for g in range(64):
    print(f"{g:5d} {us(t[g*4]):7.2f} {us(t[g*4+1]):7.2f} {us(t[g*4+2]):7.2f}")
print("tile  acc    done   released")
for l in range(16):
    print(f"{l:4d} {us(t[256+l*4]):7.2f} {us(t[256+l*4+1]):7.2f} {us(t[256+l*4+2]):7.2f}")
