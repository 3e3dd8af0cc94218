#!/bin/bash
# Mainloop ceiling (dense 8192^3 engine vs cuBLAS, bf16 + TF32) and ncu --set full
# captures of the dense engine GEMM, L14 upd, L2 fwd and the stem im2col/col2im.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python tools/probes/dense_peak.py --out gpurun_out/dense_peak.json 2>&1 | tail -6
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
timeout 600 $NCU -k regex:engine_kernel -s 1 -c 1 -o gpurun_out/r02_dense8192 -f python /tmp/dense1.py > gpurun_out/ncu_dense.log 2>&1; tail -2 gpurun_out/ncu_dense.log
timeout 600 $NCU -k regex:engine_kernel -s 1 -c 1 -o gpurun_out/r02_L14_upd -f python tools/probes/layer_once.py 14 upd 2 > gpurun_out/ncu_l14.log 2>&1; tail -2 gpurun_out/ncu_l14.log
timeout 600 $NCU -k regex:engine_kernel -s 1 -c 1 -o gpurun_out/r02_L2_fwd -f python tools/probes/layer_once.py 2 fwd 2 > gpurun_out/ncu_l2.log 2>&1; tail -2 gpurun_out/ncu_l2.log
timeout 600 $NCU -k regex:"im2col|col2im|engine_kernel" -c 8 -o gpurun_out/r02_stem -f python tools/probes/layer_once.py 1 bwd 1 > gpurun_out/ncu_stem.log 2>&1; tail -2 gpurun_out/ncu_stem.log
timeout 600 $NCU -k regex:"im2col" -c 1 -o gpurun_out/r02_stem_fwd -f python tools/probes/layer_once.py 1 fwd 1 > gpurun_out/ncu_stemf.log 2>&1; tail -2 gpurun_out/ncu_stemf.log
ls -la gpurun_out/*.ncu-rep
