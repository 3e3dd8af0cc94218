"""One m=n=k=32, batch 16 stride BRGEMM launch (1184 jobs, gather path) for an ncu capture."""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch  # noqa: E402

from paper_1906_06440_b200 import _lib  # noqa: E402

lib = _lib.load()
m = n = k = int(os.environ.get("M", "32"))
batch, jobs = 16, 1184
a = torch.randn(jobs * batch * k * m, device="cuda").bfloat16()
b = torch.randn(jobs * batch * n * k, device="cuda").bfloat16()
c = torch.empty(jobs * n * m, device="cuda")
for _ in range(3):
    _lib.check(lib.brk_brgemm_stride(a.data_ptr(), b.data_ptr(), k * m, n * k, c.data_ptr(), jobs, batch * k * m,
                                     batch * n * k, n * m, m, n, k, batch, m, k, m, 1.0, 0.0, _lib.BRK_BF16,
                                     _lib.BRK_F32, _lib.BRK_COMPUTE_BF16, 0))
torch.cuda.synchronize()
print("ok")
