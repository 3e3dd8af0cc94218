ncu --set full --import-source on --clock-control none -k regex:engine_group_kernel -s 2 -c 1 \
    --section WarpStateStats --section SourceCounters -f -o gpurun_out/mlp_group3 python tools/_probe_mlp.py > gpurun_out/ncu_mlp3.log 2>&1
tail -3 gpurun_out/ncu_mlp3.log
