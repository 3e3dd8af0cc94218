"""TMA global->smem throughput per SM: box size x issuing warps (L2-resident source, 74 CTAs)."""
import ctypes, sys
import torch
sys.path.insert(0, '.')
from paper_1906_06440_b200 import _lib
lib = _lib.load()
rows, cols = 4096, 1024
buf = torch.randn(rows, cols, device="cuda").bfloat16()
for ctas in (74, 148):
    for box in (64, 128, 256):
        for warps in (1, 2, 4, 8):
            stages = max(1, min(12, (192 * 1024) // (box * 128)))
            stages -= stages % warps if stages >= warps else 0
            if stages < warps:
                continue
            us = ctypes.c_float(); by = ctypes.c_double()
            rc = lib.brk_diag_tma_bw(buf.data_ptr(), rows, cols, box, 1, stages, ctas, 3000, warps, ctypes.byref(us),
                                     ctypes.byref(by))
            assert rc == 0, _lib.last_error()
            gbs = by.value / (us.value * 1e-6) / 1e9
            print(f"ctas {ctas:3d} box {box:3d} rows ({box*128//1024:2d} KB) warps {warps} stages {stages:2d}: "
                  f"per SM {gbs / ctas / 1.965:6.1f} B/clk  total {gbs:7.0f} GB/s", flush=True)
