J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])'
for o in b4b3u4b2u3b1u2u1 b4b3u4b2u3u2u1b1 b4b3u4b2u3u1u2b1 b4u4b3b2u3u1b1u2 b4b3u4b2u1u3u2b1 b4b3b2u4u1u3b1u2 b4b3u4b2u3u1b1u2; do
  echo -n "$o "; BRK_MLP_ORDER=$o python bench.py --steps 100 --warmup 5 2>&1 | tail -1 | python -c "$J"
done
BRK_MLP_ORDER=b4b3u4b2u3u1b1u2 python tools/_probe_mlp_ts.py 2>&1 | tail -8
