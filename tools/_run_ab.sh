python tools/_probe_stem.py 2>&1 | grep gemm_upd
P='import sys; sys.path.insert(0, "."); sys.path.insert(0, "tools"); import suites; r = suites.lstm_suite(iters=5); print(round(r["fwd"]["tflops"],1), round(r["bwd_upd"]["tflops"],1), round(r["all"]["tflops"],1))'
python -c "$P"; python -c "$P"
python -m pytest tests/test_gpu_dense.py tests/test_gpu_lstm.py tests/test_gpu_conv_small.py -q 2>&1 | tail -1
