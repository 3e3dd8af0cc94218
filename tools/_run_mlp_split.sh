for bf in 1 0 1 0; do BRK_MLP_BFIRST=$bf python bench.py --steps 50 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bfirst=$bf', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"; done
BRK_MLP_BFIRST=0 python tools/_probe_mlp_ts.py 2>&1 | tail -13
