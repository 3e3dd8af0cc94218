"""BASELINE config 1 as one launch (stride BRGEMM, m=n=k=64, batch 16, 1184 jobs, bf16 -> fp32), for ncu."""
import sys
import torch
sys.path.insert(0, '.')
from paper_1906_06440_b200 import _lib
lib = _lib.load()
m = n = k = 64; batch = 16; jobs = 1184
a = torch.randn(jobs * batch * k * m, device="cuda").bfloat16()
b = torch.randn(jobs * batch * n * k, device="cuda").bfloat16()
c = torch.empty(jobs * n * m, device="cuda")
for _ in range(3):
    _lib.check(lib.brk_brgemm_stride(a.data_ptr(), b.data_ptr(), k * m, n * k, c.data_ptr(), jobs, batch * k * m,
                                     batch * n * k, n * m, m, n, k, batch, m, k, m, 1.0, 0.0, _lib.BRK_BF16,
                                     _lib.BRK_F32, _lib.BRK_COMPUTE_BF16, None))
torch.cuda.synchronize()
