#!/bin/bash
# ncu --set full captures summarised on the box (reports are too big to bring back all).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/ncu
NCU="ncu --set full --clock-control none --import-source on"
cat > /tmp/dense1.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_1906_06440_b200 import _dense
M=N=K=8192
a=torch.randn(M,K,device="cuda").bfloat16(); b=torch.randn(N,K,device="cuda").bfloat16()
c=torch.empty(M,N,device="cuda",dtype=torch.bfloat16)
for _ in range(2): _dense.gemm(a,b,c,split=False)
torch.cuda.synchronize()
PY
cap() { name=$1; shift; timeout 600 $NCU -o /tmp/$name -f "$@" > /tmp/$name.log 2>&1; tail -1 /tmp/$name.log;
  python tools/ncu_summary.py /tmp/$name.ncu-rep > gpurun_out/ncu/$name.json; }
cap r02_dense8192 -k regex:engine_kernel -s 1 -c 1 python /tmp/dense1.py
cap r02_L14_upd -k regex:engine_kernel -s 1 -c 1 python tools/probes/layer_once.py 14 upd 2
cap r02_L2_fwd -k regex:engine_kernel -s 1 -c 1 python tools/probes/layer_once.py 2 fwd 2
cap r02_L15_upd -k regex:engine_kernel -s 1 -c 1 python tools/probes/layer_once.py 15 upd 2
cap r02_L4_fwd -k regex:engine_kernel -s 1 -c 1 python tools/probes/layer_once.py 4 fwd 2
cap r02_stem_bwd -k regex:"im2col|col2im|engine_kernel" -c 8 python tools/probes/layer_once.py 1 bwd 1
cap r02_stem_fwd -k regex:"im2col|engine_kernel" -c 4 python tools/probes/layer_once.py 1 fwd 1
cap r02_stem_upd -k regex:"im2col|engine_kernel|split_reduce" -c 6 python tools/probes/layer_once.py 1 upd 1
cp /tmp/r02_dense8192.ncu-rep /tmp/r02_L14_upd.ncu-rep gpurun_out/ncu/
ls -la gpurun_out/ncu
