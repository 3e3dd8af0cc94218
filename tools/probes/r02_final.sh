#!/bin/bash
# Final GPU pass of the round: tests, smoke, bench line, reference arm, launch list of the
# bench command (ncu, cold per-launch times) and one ncu --set full of the headline kernel.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
bash tools/probes/r02_full.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
tail -2 gpurun_out/ncu_bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_step_kernel -s 5 -c 1 \
  -o gpurun_out/r02_mlp_final -f python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_mlp.log 2>&1
tail -2 gpurun_out/ncu_mlp.log
