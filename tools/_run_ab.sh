J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["us_per_launch"])'
python -m pytest tests/test_gpu_mlp.py tests/test_gpu_fc.py -x -q 2>&1 | tail -2
for i in 1 2; do python bench.py --steps 100 --warmup 5 2>&1 | tail -1 | python -c "$J"; done
python tools/_probe_mlp.py && echo probe-ok
