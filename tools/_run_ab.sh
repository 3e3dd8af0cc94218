timeout 900 python - <<'PY'
import sys, json
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import suites
r = suites.resnet_suite(n=256, iters=5, layers=[1])
for row in r["layers"]:
    print(row["id"], row["path"], {p: (round(row[p]["us"], 1), round(row[p]["tflops"], 1), round(row[p]["roof_frac"], 3)) for p in ("fwd", "bwd", "upd")})
PY
