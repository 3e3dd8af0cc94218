python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > gpurun_out/bench_full3.json 2> gpurun_out/bench_full3.err; tail -c 300 gpurun_out/bench_full3.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_full3.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step")}, d["e2e"]["value"], d["roofline"]["achieved"], d["roofline"]["frac"], d["roofline"]["traffic"])
w = d["workloads"]
print("resnet all53", {p: round(v["tflops"], 1) for p, v in w["resnet50_conv_n256"]["summary"].items()})
print("resnet engine", {p: round(v["tflops"], 1) for p, v in w["resnet50_conv_n256"]["summary_engine_layers"].items()})
print("lstm", w["lstm_t50_n168_c1024"]["all"])
print("brgemm cfg1", w["brgemm"]["config1_stride_16x64x64x64"])
print("split", w["brgemm_vs_split_gemm"])
PY
ncu --set full --import-source on --clock-control none -k regex:engine_group_kernel -s 3 -c 1 -f -o gpurun_out/mlp_group_r01e python tools/_probe_mlp.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r01e.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
ls gpurun_out/*r01e*
