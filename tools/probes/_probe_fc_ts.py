"""In-kernel phase stamps of one brk_fc_fwd launch at the MLP shape (per CTA, slots of brk_engine.cu BRK_TS)."""
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
y32 = torch.empty(N // 64, K // 64, 64, 64, device="cuda", dtype=torch.float32)
for bias, act, bf in ((True, 1, 1), (False, 1, 1), (False, 0, 1), (False, 0, 0), (True, 1, 1)):
    out = y if bf else y32
    def call():
        assert lib.brk_fc_fwd(x.data_ptr(), w.data_ptr(), b.data_ptr() if bias else None, out.data_ptr(), N, C, K,
                              64, 64, 64, act, bf, None) == 0
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    ts = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
    lib.brk_diag_set_timestamps(ts.data_ptr())
    call(); torch.cuda.synchronize(); call()
    torch.cuda.synchronize()
    lib.brk_diag_set_timestamps(None)
    a = ts.cpu().numpy().reshape(148, 16).astype(np.int64)
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    print(f"bias={bias} act={act} bf16={bf}")
    names = {0: "entry", 1: "setup", 2: "firstTMA", 3: "firstFull", 4: "lastCommit", 5: "accReady", 8: "c0start", 9: "c0flush", 10: "c1start", 11: "c1flush", 12: "loopDone", 13: "arrived", 6: "epiDone", 7: "exit"}
    for k, n in names.items():
        v = a[:, k]
        v = v[v > 0]
        if len(v):
            print(f"{k:2d} {n:11s} median {np.median(v - t0) / 1e3:7.2f} us   min {np.min(v - t0) / 1e3:7.2f}  max {np.max(v - t0) / 1e3:7.2f}")
