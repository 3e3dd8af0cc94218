J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])'
python -m pytest tests/test_gpu_mlp.py -x -q 2>&1 | tail -2
for i in 1 2; do
for w in 0 1; do echo -n "whole=$w "; BRK_MLP_UPD_WHOLE=$w python bench.py --steps 100 --warmup 5 2>&1 | tail -1 | python -c "$J"; done
done
python tools/_probe_mlp_ts.py 2>&1 | tail -8
