python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -1 gpurun_out/bench_full.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r01c.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:engine_group_kernel -s 3 -c 1 -f -o gpurun_out/mlp_group_r01c python tools/_probe_mlp.py > /dev/null 2>&1
ls -la gpurun_out/ | tail -5
