"""Weight-update tile / split sweep for selected ResNet-50 layers (BRK_CONV_TILE / BRK_CONV_SPLITS)."""
import ctypes
import os
import subprocess
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tools')
layers = [int(x) for x in sys.argv[1].split(",")]
if os.environ.get("CHILD"):
    import suites
    from paper_1906_06440_b200 import _lib
    lib = _lib.load()
    r = suites.resnet_suite(n=256, iters=5, layers=layers, passes=("upd",))
    for row in r["layers"]:
        g = (256, row["C"], row["K"], row["H"], row["W"], row["R"], row["R"], row["stride"], row["R"] // 2, row["R"] // 2)
        out = (ctypes.c_int * 3)()
        lib.brk_conv_plan(2, *g, out)
        print(os.environ.get("BRK_CONV_TILE", "-"), os.environ.get("BRK_CONV_SPLITS", "-"), row["id"],
              round(row["upd"]["us"], 1), round(row["upd"]["roof_frac"], 3), list(out), flush=True)
    sys.exit(0)
for tile in (None, "1,256", "1,128"):
    for sp in (None, "4", "8", "16", "32", "64"):
        env = dict(os.environ, CHILD="1")
        if tile: env["BRK_CONV_TILE"] = tile
        if sp: env["BRK_CONV_SPLITS"] = sp
        subprocess.run([sys.executable, __file__, sys.argv[1]], env=env)
