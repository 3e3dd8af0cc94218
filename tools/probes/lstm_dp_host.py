"""Host-side profile of LstmDP.step (cProfile over 10 steps after warm-up)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch  # noqa: E402

from paper_1906_06440_b200.train import LstmDP  # noqa: E402

net = LstmDP()
for _ in range(3):
    net.step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    net.step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {((t1 - t0) / 10) * 1e3:.3f} ms/step, wall {((t2 - t0) / 10) * 1e3:.3f} ms/step")
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    net.step()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
