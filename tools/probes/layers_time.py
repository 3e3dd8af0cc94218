"""Time selected ResNet-50 layers (N=256, all passes) via tools/suites.resnet_suite.
    python tools/probes/layers_time.py 2 4 14
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from tools.suites import resnet_suite  # noqa: E402

ids = [int(a) for a in sys.argv[1:]] or [2]
res = resnet_suite(n=256, iters=5, layers=ids)
for r in res["layers"]:
    print(f"L{r['id']:2d} {r['path']:11s}", {p: (round(r[p]["us"], 1), round(r[p]["roof_frac"], 3)) for p in ("fwd", "bwd", "upd") if r.get(p)},
          r.get("plan"), flush=True)
