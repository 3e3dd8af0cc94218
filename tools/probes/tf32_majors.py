"""TF32 engine: every (A, B) major combination at a few shapes; prints the error of each."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch  # noqa: E402

from paper_1906_06440_b200._dense import gemm  # noqa: E402

torch.manual_seed(0)
for (m, n, k) in [(256, 256, 256), (256, 256, 64), (128, 128, 32), (384, 512, 1000), (256, 512, 128)]:
    for a_t in (False, True):
        for b_t in (False, True):
            for dt in (torch.float32, torch.bfloat16):
                a = torch.randint(-3, 4, (k, m) if a_t else (m, k), device="cuda").to(dt)
                b = torch.randint(-3, 4, (k, n) if b_t else (n, k), device="cuda").to(dt)
                out = torch.zeros(m, n, device="cuda")
                try:
                    gemm(a, b, out, a_t=a_t, b_t=b_t, split=False)
                    am = (a.t() if a_t else a).double()
                    bm = (b.t() if b_t else b).double()
                    ref = am @ bm.t()
                    err = (out.double() - ref).abs().max().item()
                    print(f"{m}x{n}x{k} a_t={a_t:d} b_t={b_t:d} {str(dt)[6:]:9s} maxabs err {err:.3g} "
                          f"nonzero {int((out != 0).sum())}/{out.numel()}", flush=True)
                except Exception as exc:  # noqa: BLE001
                    print(f"{m}x{n}x{k} a_t={a_t:d} b_t={b_t:d} {dt}: {exc}", flush=True)
