"""Epilogue chunk loop run twice per tile (BRK_DEBUG_FLAGS bit 128): cold vs warm i-cache timing."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1906_06440_b200 import _lib
lib = _lib.load()
N, C, K = 2048, 1024, 1024
x = torch.randn(N // 64, C // 64, 64, 64, device="cuda").bfloat16()
w = torch.randn(K // 64, C // 64, 64, 64, device="cuda").bfloat16()
y = torch.empty(N // 64, K // 64, 64, 64, device="cuda", dtype=torch.bfloat16)
b = torch.randn(K, device="cuda")
for flags in ("128", "192"):
    os.environ["BRK_DEBUG_FLAGS"] = flags
    def call():
        assert lib.brk_fc_fwd(x.data_ptr(), w.data_ptr(), b.data_ptr(), y.data_ptr(), N, C, K, 64, 64, 64, 1, 1, None) == 0
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    ts = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
    lib.brk_diag_set_timestamps(ts.data_ptr())
    call()
    torch.cuda.synchronize()
    lib.brk_diag_set_timestamps(None)
    a = ts.cpu().numpy().reshape(148, 16).astype(np.int64)
    a = a[a[:, 0] > 0]
    print(f"flags={flags}: pass 1 (cold) {np.median(a[:, 14] - a[:, 5]) / 1e3:.2f} us, "
          f"pass 2 (warm) {np.median(a[:, 15] - a[:, 14]) / 1e3:.2f} us")
    m = lambda i, j: np.median(a[:, j] - a[:, i]) / 1e3  # noqa: E731
    print(f"   warm: ->c0 {m(14, 8):.2f}  c0 stage {m(8, 10):.2f}  c1 stage {m(10, 11):.2f}  flush {m(11, 15):.2f}")
