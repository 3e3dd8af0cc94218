python -m pytest tests/test_gpu_brgemm_tma.py tests/test_gpu_brgemm.py -x -q 2>&1 | tail -2
timeout 300 python - <<'PY'
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import suites
r = suites.brgemm_suite(ms=(64, 128, 256), batches=(1, 16, 64), variants=("stride", "offset"))
for p in r["points"]:
    print(p["m"], p["batch"], p["variant"], p["jobs"], round(p["us"], 1), round(p["tflops"], 2), round(p["roof_frac"], 3))
PY
