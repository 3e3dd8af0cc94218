"""Stem conv (C=3, 7x7/2, N=256) on the small-channel path: per-kernel device times."""
import sys
import torch
sys.path.insert(0, '.')
from paper_1906_06440_b200 import _lib
from paper_1906_06440_b200._dense import gemm
lib = _lib.load()
n, c, h, w, r, s, st, pad = 256, 3, 224, 224, 7, 7, 2, 3
p = q = 112
rsc, ld = r * s * c, 192
pix = n * p * q
x = torch.randn(n, 1, h, w, c, device="cuda").bfloat16()
col = torch.empty(pix, ld, device="cuda", dtype=torch.bfloat16)
col152 = torch.empty(pix, 152, device="cuda", dtype=torch.bfloat16)
w2 = torch.randn(64, ld, device="cuda").bfloat16()
out = torch.empty(pix, 64, device="cuda", dtype=torch.bfloat16)
do = torch.randn(pix, 64, device="cuda").bfloat16()
dwt = torch.empty(rsc, 64, device="cuda")
dcol = torch.empty(pix, ld, device="cuda", dtype=torch.bfloat16)
col152 = torch.empty(pix, 152, device="cuda", dtype=torch.bfloat16)
dx = torch.empty(n, 1, h, w, c, device="cuda", dtype=torch.bfloat16)
ops = {
    "im2col": lambda: lib.brk_conv_im2col(x.data_ptr(), col.data_ptr(), n, c, h, w, r, s, st, pad, pad, c, ld, None),
    "im2col152": lambda: lib.brk_conv_im2col(x.data_ptr(), col152.data_ptr(), n, c, h, w, r, s, st, pad, pad, c, 152,
                                             None),
    "gemm_fwd152": lambda: gemm(col152[:, :rsc], w2[:, :rsc], out),
    "gemm_fwd": lambda: gemm(col[:, :rsc], w2[:, :rsc], out),
    "gemm_upd": lambda: gemm(col[:, :rsc], do, dwt, a_t=True, b_t=True),
    "gemm_bwd": lambda: gemm(do, w2, dcol, b_t=True),
    "col2im": lambda: lib.brk_conv_col2im(dcol.data_ptr(), dx.data_ptr(), n, c, h, w, r, s, st, pad, pad, c, ld, None),
}
for name, fn in ops.items():
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:9s} {e0.elapsed_time(e1) / 5 * 1e3:9.1f} us")
