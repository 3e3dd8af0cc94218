P='import sys; sys.path.insert(0, "."); sys.path.insert(0, "tools"); import suites; r = suites.lstm_suite(iters=5); print(round(r["fwd"]["tflops"],1), round(r["bwd_upd"]["tflops"],1), round(r["all"]["tflops"],1))'
python -m pytest tests/test_gpu_lstm.py -x -q 2>&1 | tail -2
for i in 1 2; do echo -n "new "; python -c "$P" 2>&1 | tail -1; echo -n "full "; BRK_LSTM_FULL_TILE=1 python -c "$P" 2>&1 | tail -1; done
python tools/_probe_lstm_ts.py 2>&1 | tail -7
