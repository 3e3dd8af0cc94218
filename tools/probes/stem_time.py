"""Time the ResNet-50 stem (N=256, 3->64, 7x7/2) passes through the conv API on the GPU:
CUDA events, L2 flushed, both small-channel paths (BRK_CONV_S2D=1 / 0)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch  # noqa: E402

from tools.suites import resnet_suite  # noqa: E402

for mode in ("1", "0"):
    os.environ["BRK_CONV_S2D"] = mode
    r = resnet_suite(n=256, iters=5, layers=[1])["layers"][0]
    print("s2d" if mode == "1" else "im2col", r["path"],
          {p: (round(r[p]["us"], 1), round(r[p]["roof_frac"], 3)) for p in ("fwd", "bwd", "upd")}, flush=True)
