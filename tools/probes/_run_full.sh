python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > gpurun_out/bench_full5.json 2> gpurun_out/bench_full5.err; tail -c 300 gpurun_out/bench_full5.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_full5.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step")}, d["e2e"]["value"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"])
w = d["workloads"]
print("resnet all53", {p: round(v["tflops"], 1) for p, v in w["resnet50_conv_n256"]["summary"].items()})
print("resnet engine", {p: round(v["tflops"], 1) for p, v in w["resnet50_conv_n256"]["summary_engine_layers"].items()})
print("stem", w["resnet50_conv_n256"]["per_layer_us"].get("1") or w["resnet50_conv_n256"]["per_layer_us"].get(1))
print("lstm", w["lstm_t50_n168_c1024"]["all"])
print("brgemm cfg1", w["brgemm"]["config1_stride_16x64x64x64"])
PY
