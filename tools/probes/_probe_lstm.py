"""Run one LSTM fwd+bwd at the benchmark config (for ncu launch lists)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1906_06440_b200 import precision
from paper_1906_06440_b200.lstm import LstmCellWeights, LstmParams, lstm_backward, lstm_forward
T, N, C, K = 50, 168, 1024, 1024
rng = np.random.default_rng(0)
params = LstmParams.from_dense(LstmCellWeights.random(rng, C, K), T, N)
x = torch.from_numpy(rng.uniform(-1, 1, (T, N, C)).astype(np.float32)).cuda()
dh = torch.from_numpy(rng.uniform(-1, 1, (T, N, K)).astype(np.float32)).cuda()
with precision("bf16"):
    for _ in range(2):
        seq = lstm_forward(params, x)
        g = lstm_backward(params, x, seq, dh)
torch.cuda.synchronize()
