"""Engine mainloop ceiling: brk_gemm_dense at 8192^3 bf16 (and a few other shapes)
against torch.matmul (cuBLAS) bf16 and TF32 on the same GPU.  Prints one JSON line.

Usage (GPU box):  python tools/probes/dense_peak.py [--out gpurun_out/dense_peak.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch  # noqa: E402

from paper_1906_06440_b200 import _dense  # noqa: E402


def timed(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(iters):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--shapes", default="8192x8192x8192,4096x4096x4096,2048x1024x1024,16384x1024x1024")
    args = ap.parse_args()
    torch.manual_seed(0)
    res = {}
    for sh in args.shapes.split(","):
        M, N, K = (int(v) for v in sh.split("x"))
        a = torch.randn(M, K, device="cuda").bfloat16()
        b = torch.randn(N, K, device="cuda").bfloat16()
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * M * N * K
        t_eng = timed(lambda: _dense.gemm(a, b, c, split=False))
        ref = (a.float() @ b.float().t())
        err = ((c.float() - ref).abs().max() / ref.abs().max()).item()
        t_cub = timed(lambda: torch.matmul(a, b.t(), out=c))
        row = {"engine_tflops": fl / t_eng / 1e12, "cublas_bf16_tflops": fl / t_cub / 1e12, "engine_err": err}
        if M == N == K == 8192:
            af, bf = a.float(), b.float()
            cf = torch.empty(M, N, device="cuda")
            from paper_1906_06440_b200 import _lib
            from paper_1906_06440_b200._device import stream_ptr
            lib = _lib.load()
            # engine TF32 on pre-rounded fp32 operands (rounding passes excluded: kernel ceiling)
            t_e32 = timed(lambda: _lib.check(lib.brk_gemm_dense_f32(
                af.data_ptr(), K, 1, bf.data_ptr(), K, 1, cf.data_ptr(), N, 0, M, N, K, 1.0, 0.0, None, 0,
                None, 0, stream_ptr())), iters=10)
            row["engine_tf32_tflops"] = fl / t_e32 / 1e12
            torch.backends.cuda.matmul.allow_tf32 = True
            t_tf = timed(lambda: torch.matmul(af, bf.t(), out=cf), iters=10)
            torch.backends.cuda.matmul.allow_tf32 = False
            row["cublas_tf32_tflops"] = fl / t_tf / 1e12
        res[sh] = row
        print(sh, json.dumps(row), flush=True)
        del a, b, c
    line = json.dumps({"dense_peak": res})
    print(line)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
