"""Run ONE ResNet-50 conv layer pass (N=256, bf16, engine / stem path) a few times —
the target of a single-kernel ncu capture.  Usage:

    python tools/probes/layer_once.py <layer id> <fwd|bwd|upd> [reps]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch  # noqa: E402

from paper_1906_06440_b200 import _lib  # noqa: E402
from paper_1906_06440_b200.cnn import (  # noqa: E402
    ConvSpec,
    conv2d_backward_data,
    conv2d_forward,
    conv2d_weight_update,
)
from paper_1906_06440_b200.tensor import BlockedTensor  # noqa: E402
from paper_1906_06440_b200.train import RESNET50_ROWS  # noqa: E402


def main():
    lid, pas = int(sys.argv[1]), sys.argv[2]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    _, c, k, h, w, r, s, st, _ = [row for row in RESNET50_ROWS if row[0] == lid][0]
    n = 256
    spec = ConvSpec(n=n, c=c, k=k, h=h, w=w, r=r, s=s, stride=st)
    bc, bk = spec.b_c, spec.b_k
    g = torch.Generator(device="cuda").manual_seed(0)
    x = (torch.rand((n, c // bc, h, w, bc), generator=g, device="cuda") * 2 - 1).bfloat16()
    wt = ((torch.rand((k // bk, c // bc, r, s, bc, bk), generator=g, device="cuda") * 2 - 1) * 0.05).bfloat16()
    do = (torch.rand((n, k // bk, spec.out_h, spec.out_w, bk), generator=g, device="cuda") * 2 - 1).bfloat16()
    xi = BlockedTensor(x, 4, {"n": 0, "c": (1, 4), "h": 2, "w": 3})
    wi = BlockedTensor(wt, 4, {"k": (0, 5), "c": (1, 4), "r": 2, "s": 3})
    di = BlockedTensor(do, 4, {"n": 0, "k": (1, 4), "p": 2, "q": 3})
    fn = {"fwd": lambda: conv2d_forward(spec, xi, wi), "bwd": lambda: conv2d_backward_data(spec, di, wi),
          "upd": lambda: conv2d_weight_update(spec, xi, di)}[pas]
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(f"L{lid} {pas}: {reps} runs, {_lib.launch_count()} native launches")


if __name__ == "__main__":
    main()
