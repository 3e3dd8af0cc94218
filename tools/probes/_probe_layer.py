"""Debug probe: run one ResNet layer's conv passes once each with a sync after each."""
import ctypes, sys, time
import torch
sys.path.insert(0, '.')
from paper_1906_06440_b200 import _lib
from tools.suites import RESNET50_ROWS
lib = _lib.load()
lid = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
row = [r for r in RESNET50_ROWS if r[0] == lid][0]
_, c, k, h, w, r, s, st, _ = row
pad = (r - 1) // 2
p = (h + 2 * pad - r) // st + 1
geom = (n, c, k, h, w, r, s, st, pad, pad)
x = torch.randn(n, c // 64, h, w, 64, device='cuda').bfloat16()
wt = torch.randn(k // 64, c // 64, r, s, 64, 64, device='cuda').bfloat16()
do = torch.randn(n, k // 64, p, p, 64, device='cuda').bfloat16()
out = torch.empty(n, k // 64, p, p, 64, device='cuda', dtype=torch.bfloat16)
din = torch.empty_like(x)
dw = torch.empty(k // 64, c // 64, r, s, 64, 64, device='cuda')
for ps in range(3):
    o = (ctypes.c_int * 3)(); lib.brk_conv_plan(ps, *geom, o); print('plan', ps, list(o), flush=True)
nb = lib.brk_conv_upd_workspace(*geom); ws = torch.empty(max(nb, 16), dtype=torch.uint8, device='cuda')
sp = torch.cuda.current_stream().cuda_stream
passes = sys.argv[3].split(',') if len(sys.argv) > 3 else ['fwd', 'bwd', 'upd']
fns = {'fwd': lambda: lib.brk_conv_fwd(x.data_ptr(), wt.data_ptr(), None, out.data_ptr(), *geom, 64, 64, 0, 1, sp),
       'bwd': lambda: lib.brk_conv_bwd_data(do.data_ptr(), wt.data_ptr(), din.data_ptr(), *geom, 64, 64, 1, sp),
       'upd': lambda: lib.brk_conv_upd(x.data_ptr(), do.data_ptr(), dw.data_ptr(), None, 0.0, ws.data_ptr(), nb,
                                       *geom, 64, 64, 1, sp)}
for name in passes:
    t = time.time(); rc = fns[name](); torch.cuda.synchronize(); print(name, rc, time.time() - t, flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fns[name]()
    e1.record(); torch.cuda.synchronize()
    print(f"{name} {e0.elapsed_time(e1) / 20 * 1e3:.1f} us (L2-warm back-to-back)", flush=True)
