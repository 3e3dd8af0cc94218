"""Back-to-back graph replays of the fused MLP step (the bench warm-up pattern): N steps, then sync."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch  # noqa: E402

from paper_1906_06440_b200.mlp import MLP  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
m = MLP(layers=4, width=1024, batch=2048, lr=1e-4, seed=0)
g = torch.Generator(device="cuda").manual_seed(1)
m.load_input((torch.rand(m.y[0].shape, generator=g, device="cuda") * 2 - 1).bfloat16(),
             (torch.rand(m.dy.shape, generator=g, device="cuda") * 2 - 1).bfloat16())
m.capture()
torch.cuda.synchronize()
t0 = time.time()
done = 0
while done < steps:
    for _ in range(100):
        m.replay()
    done += 100
    every = int(os.environ.get("STRESS_EVERY", "1000"))
    if done % every == 0:
        torch.cuda.synchronize()
        print(f"{done} steps ok ({time.time() - t0:.2f} s)", flush=True)
torch.cuda.synchronize()
print("stress ok", os.environ.get("BRK_MLP_CHUNK"), flush=True)
