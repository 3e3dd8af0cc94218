ncu --set full --import-source on --clock-control none -k regex:engine_group_kernel -s 3 -c 1 -f -o gpurun_out/mlp_group_r01d python tools/_probe_mlp.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:brgemm_generic -s 2 -c 1 -f -o gpurun_out/brgemm_cfg1_r01d python tools/_probe_brgemm_cfg1.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r01d.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
ls -la gpurun_out/*r01d*
