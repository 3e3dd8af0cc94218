"""Forward / backward-data tile sweep over the engine ResNet-50 layers (BRK_CONV_TILE)."""
import ctypes
import json
import os
import subprocess
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tools')
if os.environ.get("CHILD"):
    import suites
    from paper_1906_06440_b200 import _lib
    lib = _lib.load()
    out = {}
    for lid in range(2, 21):
        for p in ("fwd", "bwd"):
            try:
                r = suites.resnet_suite(n=256, iters=5, layers=[lid], passes=(p,))
                row = r["layers"][0]
                out.setdefault(str(lid), {})[p] = round(row[p]["us"], 1)
                out[str(lid)].setdefault("plan", row.get("plan"))
            except Exception:  # noqa: BLE001 - the forced tile does not fit this layer
                pass
    print("RESULT", os.environ.get("BRK_CONV_TILE", "-"), json.dumps(out), flush=True)
    sys.exit(0)
for tile in (None, "1,256", "1,128", "0,256", "0,128", "0,64"):
    env = dict(os.environ, CHILD="1")
    if tile:
        env["BRK_CONV_TILE"] = tile
    subprocess.run([sys.executable, __file__], env=env)
