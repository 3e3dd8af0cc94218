J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["us_per_launch"])'
python -m pytest tests/test_gpu_mlp.py tests/test_gpu_fc.py -x -q 2>&1 | tail -1
for i in 1 2; do for w in 1 0; do echo -n "warm=$w "; BRK_MLP_WARM=$w python bench.py --steps 100 --warmup 5 2>&1 | tail -1 | python -c "$J"; done; done
python tools/_probe_mlp_ts.py 2>&1 | grep -E "fwd|bwd4"
