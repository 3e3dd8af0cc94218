"""Per-launch time of brk_fc_fwd at the MLP shape under BRK_DEBUG_FLAGS (graph of 20 launches)."""
import os, sys
import torch
sys.path.insert(0, '.')
from paper_1906_06440_b200 import _lib
lib = _lib.load()
N = C = K = 1024
N = 2048
x = torch.randn(N // 64, C // 64, 64, 64, device="cuda").bfloat16()
w = torch.randn(K // 64, C // 64, 64, 64, device="cuda").bfloat16()
y = torch.empty(N // 64, K // 64, 64, 64, device="cuda", dtype=torch.bfloat16)
b = torch.randn(K, device="cuda")
s = torch.cuda.Stream()
def call():
    assert lib.brk_fc_fwd(x.data_ptr(), w.data_ptr(), b.data_ptr(), y.data_ptr(), N, C, K, 64, 64, 64, 1, 1, s.cuda_stream) == 0
with torch.cuda.stream(s):
    call()
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for _ in range(20):
        call()
with torch.cuda.stream(s):
    g.replay(); g.replay()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5):
        g.replay()
    e1.record(s)
e1.synchronize()
print(f"flags {os.environ.get('BRK_DEBUG_FLAGS', '0')}: {e0.elapsed_time(e1) / 100 * 1e3:.2f} us per launch")
