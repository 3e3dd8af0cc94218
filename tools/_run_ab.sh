timeout 900 python - <<'PY'
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import suites
r = suites.resnet_suite(n=256, iters=5, layers=list(range(2, 21)), passes=("upd",))
print("summary", r["summary_engine_layers"]["upd"])
for row in r["layers"]:
    print(row["id"], round(row["upd"]["us"], 1), round(row["upd"]["roof_frac"], 3), row.get("plan", {}).get("upd"))
PY
