"""Per-step phase timestamps of the LSTM sequence kernels (CTA 0)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1906_06440_b200 import _lib, precision
from paper_1906_06440_b200.lstm import LstmCellWeights, LstmParams, lstm_backward, lstm_forward
T, N, C, K = 50, 168, 1024, 1024
rng = np.random.default_rng(0)
params = LstmParams.from_dense(LstmCellWeights.random(rng, C, K), T, N)
x = torch.from_numpy(rng.uniform(-1, 1, (T, N, C)).astype(np.float32)).cuda()
dh = torch.from_numpy(rng.uniform(-1, 1, (T, N, K)).astype(np.float32)).cuda()
lib = _lib.load()
ts = torch.zeros(T * 8, dtype=torch.int64, device="cuda")
tb = torch.zeros(T * 8, dtype=torch.int64, device="cuda")
with precision("bf16"):
    seq = lstm_forward(params, x)
    lstm_backward(params, x, seq, dh)
    torch.cuda.synchronize()
    lib.brk_diag_lstm_timestamps(ts.data_ptr())
    seq = lstm_forward(params, x)
    torch.cuda.synchronize()
    lib.brk_diag_lstm_timestamps(tb.data_ptr())
    lstm_backward(params, x, seq, dh)
    torch.cuda.synchronize()
    lib.brk_diag_lstm_timestamps(None)
b = tb.cpu().numpy().reshape(T, 8).astype(np.int64)[: T - 1]
print("bwd: mean step us", np.diff(b[:, 6]).mean() / 1e3)
bn = ["rel0", "relLast", "land0", "landLast", "tfull", "pready", "released"]
for i in range(1, 7):
    print(f"  {bn[i-1]}->{bn[i]}: {np.mean(b[1:, i] - b[1:, i-1]) / 1e3:.2f} us")
print(f"  released->rel0(next): {np.mean(b[1:, 0] - b[:-1, 6]) / 1e3:.2f} us")
a = ts.cpu().numpy().reshape(T, 8).astype(np.int64)
names = ["rel0", "relLast", "land0", "landLast", "accReady", "epiDone"]
t0 = a[0, 2]
print("step", " ".join(f"{n:>9s}" for n in names))
for t in range(0, T, 7):
    print(f"{t:4d}", " ".join(f"{(a[t, i] - t0) / 1e3:9.2f}" for i in range(6)))
d = np.diff(a[:, 5])
print("mean step us", d.mean() / 1e3)
for i, n in enumerate(names):
    if i == 0: continue
    print(f"  {names[i-1]}->{n}: {np.mean(a[1:, i] - a[1:, i-1]) / 1e3:.2f} us")
print(f"  epiDone->rel0(next): {np.mean(a[1:, 0] - a[:-1, 5]) / 1e3:.2f} us")
