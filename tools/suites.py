"""Device-timed workload suites used by bench.py (and runnable alone):

* ``resnet_suite``  — the 20 ResNet-50 convolution shapes of the reference's
  bench table (pkg/src/brkernels/bench.py:57-79, occurrence counts n_i summing
  to 53) at minibatch N, fwd / bwd-data / weight update, with the reference's
  weighted efficiency  sum(n_i F_i) / sum(n_i t_i) / peak  (bench.py:142-152).
* ``lstm_suite``    — the LSTM cell C=K=1024, N=168, T=50 fwd and bwd+upd.

Timing: every launch is bracketed by CUDA events on the launching stream with
an L2 flush (a 256 MiB write) between launches, outside the events.

    python tools/suites.py conv [N]      python tools/suites.py lstm
"""

from __future__ import annotations

import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

# (id, C, K, H, W, R, S, stride, count) — reference bench.py:57-79
RESNET50_ROWS = (
    (1, 3, 64, 224, 224, 7, 7, 2, 1),
    (2, 64, 256, 56, 56, 1, 1, 1, 4),
    (3, 64, 64, 56, 56, 1, 1, 1, 1),
    (4, 64, 64, 56, 56, 3, 3, 1, 3),
    (5, 256, 64, 56, 56, 1, 1, 1, 2),
    (6, 256, 512, 56, 56, 1, 1, 2, 1),
    (7, 256, 128, 56, 56, 1, 1, 2, 1),
    (8, 128, 128, 28, 28, 3, 3, 1, 4),
    (9, 128, 512, 28, 28, 1, 1, 1, 4),
    (10, 512, 128, 28, 28, 1, 1, 1, 3),
    (11, 512, 1024, 28, 28, 1, 1, 2, 1),
    (12, 512, 256, 28, 28, 1, 1, 2, 1),
    (13, 256, 256, 14, 14, 3, 3, 1, 6),
    (14, 256, 1024, 14, 14, 1, 1, 1, 6),
    (15, 1024, 256, 14, 14, 1, 1, 1, 5),
    (16, 1024, 2048, 14, 14, 1, 1, 2, 1),
    (17, 1024, 512, 14, 14, 1, 1, 2, 1),
    (18, 512, 512, 7, 7, 3, 3, 1, 3),
    (19, 512, 2048, 7, 7, 1, 1, 1, 3),
    (20, 2048, 512, 7, 7, 1, 1, 1, 2),
)


def _peaks():
    try:
        pk = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return pk["bf16_tflops"], pk["hbm_gbs"], "measured"
    except (OSError, ValueError, KeyError):
        return 1590.0, 6650.0, "fallback"


class _Timer:
    def __init__(self, torch):
        self.torch = torch
        self.flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def __call__(self, fn, iters, warmup=2):
        torch = self.torch
        stream = torch.cuda.current_stream()
        for _ in range(warmup):
            fn(stream.cuda_stream)
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        for i in range(iters):
            self.flush.fill_(float(i))
            evs[i][0].record(stream)
            fn(stream.cuda_stream)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        ts = [a.elapsed_time(b) * 1e-3 for a, b in evs]
        return statistics.fmean(ts), min(ts)


def resnet_suite(n=256, iters=10, layers=None, passes=("fwd", "bwd", "upd"), verbose=False, precision="bf16"):
    """Per-layer device time of the conv passes at minibatch n (64-channel blocks): bf16 storage,
    or fp32 storage with TF32 math (precision="tf32", roofline against the TF32 peak)."""
    import torch

    from paper_1906_06440_b200 import _lib
    from paper_1906_06440_b200.cnn import ConvSpec, conv2d_backward_data, conv2d_forward, conv2d_weight_update
    from paper_1906_06440_b200.tensor import BlockedTensor

    lib = _lib.load()
    peak, hbm, src = _peaks()
    tf32 = precision == "tf32"
    if tf32:
        peak = _tf32_peak(peak)
    dt = torch.float32 if tf32 else torch.bfloat16
    code = _lib.BRK_F32 if tf32 else _lib.BRK_BF16
    timer = _Timer(torch)
    rows = []
    tot = {p: [0.0, 0.0, 0.0] for p in passes}  # sum n_i F_i, sum n_i t_i, sum n_i t_roof
    tot_engine = {p: [0.0, 0.0, 0.0] for p in passes}  # the same over the implicit-GEMM engine layers
    g = torch.Generator(device="cuda").manual_seed(0)
    for lid, c, k, h, w, r, s, st, cnt in RESNET50_ROWS:
        if layers and lid not in layers:
            continue
        t_layer = time.time()
        spec = ConvSpec(n=n, c=c, k=k, h=h, w=w, r=r, s=s, stride=st)
        p_, q_ = spec.out_h, spec.out_w
        bc, bk = spec.b_c, spec.b_k
        geom = (n, c, k, h, w, r, s, st, spec.pad_h, spec.pad_w)
        x = (torch.rand((n, c // bc, h, w, bc), generator=g, device="cuda") * 2 - 1).to(dt)
        wt = ((torch.rand((k // bk, c // bc, r, s, bc, bk), generator=g, device="cuda") * 2 - 1) * 0.05).to(dt)
        dout = (torch.rand((n, k // bk, p_, q_, bk), generator=g, device="cuda") * 2 - 1).to(dt)
        flops = 2.0 * n * k * c * r * s * p_ * q_
        e = 4 if tf32 else 2
        act_in, act_out, wbytes = n * c * h * w * e, n * k * p_ * q_ * e, k * c * r * s * e
        # a 1x1 strided conv reads only the sampled input pixels (one in stride^2) in fwd / upd;
        # bwd-data writes the whole input gradient (the skipped pixels get zeros)
        act_read = n * c * p_ * q_ * e if (r == 1 and s == 1 and st > 1) else act_in
        bytes_ = {"fwd": act_read + wbytes + act_out, "bwd": act_out + wbytes + act_in,
                  "upd": act_read + act_out + k * c * r * s * 4}
        engine = bc == 64 and bk == 64
        calls = {}
        if engine:
            out = torch.empty((n, k // 64, p_, q_, 64), dtype=dt, device="cuda")
            din = torch.empty_like(x)
            dw = torch.empty((k // 64, c // 64, r, s, 64, 64), dtype=torch.float32, device="cuda")
            nbytes = lib.brk_conv_upd_workspace(*geom)
            ws = torch.empty(max(nbytes, 16), dtype=torch.uint8, device="cuda")
            calls["fwd"] = lambda sp: _lib.check(lib.brk_conv_fwd(x.data_ptr(), wt.data_ptr(), None, out.data_ptr(),
                                                                  *geom, 64, 64, 0, code, sp))
            calls["bwd"] = lambda sp: _lib.check(lib.brk_conv_bwd_data(dout.data_ptr(), wt.data_ptr(), din.data_ptr(),
                                                                       *geom, 64, 64, code, sp))
            calls["upd"] = lambda sp: _lib.check(lib.brk_conv_upd(x.data_ptr(), dout.data_ptr(), dw.data_ptr(), None,
                                                                  0.0, ws.data_ptr() if nbytes else None, nbytes,
                                                                  *geom, 64, 64, code, sp))
            path = "engine"
        else:
            xi = BlockedTensor(x, 4, {"n": 0, "c": (1, 4), "h": 2, "w": 3})
            wi = BlockedTensor(wt, 4, {"k": (0, 5), "c": (1, 4), "r": 2, "s": 3})
            do = BlockedTensor(dout, 4, {"n": 0, "k": (1, 4), "p": 2, "q": 3})
            calls["fwd"] = lambda sp: conv2d_forward(spec, xi, wi, precision=precision)
            calls["bwd"] = lambda sp: conv2d_backward_data(spec, do, wi, precision=precision)
            calls["upd"] = lambda sp: conv2d_weight_update(spec, xi, do, precision=precision)
            path = ("s2d-engine" if st == 2 and c <= 4 else "im2col-gemm") if c < 64 and k == 64 else "grouped"
        row = {"id": lid, "count": cnt, "path": path, "C": c, "K": k, "H": h, "W": w, "R": r, "stride": st,
               "gflop": flops / 1e9}
        for p in passes:
            if p not in calls:
                row[p] = None
                continue
            mean, best = timer(calls[p], iters)
            t_roof = max(flops / (peak * 1e12), bytes_[p] / (hbm * 1e9))
            row[p] = {"us": mean * 1e6, "us_min": best * 1e6, "tflops": flops / mean / 1e12,
                      "roof_frac": t_roof / mean, "gbs": bytes_[p] / mean / 1e9,
                      "bound": "tensor" if flops / (peak * 1e12) >= bytes_[p] / (hbm * 1e9) else "hbm"}
            if p == "bwd" and lid == 1:
                continue
            for tt in (tot, tot_engine) if engine else (tot,):
                tt[p][0] += cnt * flops
                tt[p][1] += cnt * mean
                tt[p][2] += cnt * t_roof
        if engine:
            row["plan"] = {pn: list(_plan(lib, i, geom)) for i, pn in enumerate(("fwd", "bwd", "upd"))}
        row["wall_s"] = round(time.time() - t_layer, 2)
        rows.append(row)
        if verbose:
            print(json.dumps(row), flush=True)
        del x, wt, dout
        torch.cuda.empty_cache()
    def summarize(totals):
        out = {}
        for p, (f, t, tr) in totals.items():
            if t > 0:
                out[p] = {"tflops": f / t / 1e12, "weighted_eff_vs_peak": f / t / (peak * 1e12),
                          "frac_of_roofline": tr / t, "ms": t * 1e3}
        F = sum(v[0] for v in totals.values())
        T = sum(v[1] for v in totals.values())
        TR = sum(v[2] for v in totals.values())
        if T > 0:
            out["all"] = {"tflops": F / T / 1e12, "weighted_eff_vs_peak": F / T / (peak * 1e12),
                          "frac_of_roofline": TR / T, "ms": T * 1e3, "gflop": F / 1e9}
        return out

    return {"n": n, "precision": precision, "peak_tflops": peak, "hbm_gbs": hbm, "peak_source": src, "layers": rows,
            "summary": summarize(tot), "summary_engine_layers": summarize(tot_engine)}


def lstm_suite(t_steps=50, n=168, c=1024, k=1024, iters=3, precision="bf16"):
    """LSTM cell (BASELINE config 3): fwd and bwd+upd device time at T steps.

    FLOPs as the reference (bench.py:97-103): fwd 2TN(4KC+4KK); bwd+upd twice that.
    """
    import numpy as np
    import torch

    from paper_1906_06440_b200 import precision as prec_ctx
    from paper_1906_06440_b200.lstm import LstmCellWeights, LstmParams, lstm_backward, lstm_forward

    rng = np.random.default_rng([0, 303])
    wt = LstmCellWeights.random(rng, c, k)
    params = LstmParams.from_dense(wt, t_steps, n)
    x = torch.from_numpy(rng.uniform(-1, 1, (t_steps, n, c)).astype(np.float32)).cuda()
    dh = torch.from_numpy(rng.uniform(-1, 1, (t_steps, n, k)).astype(np.float32)).cuda()
    flops_fwd = 2.0 * t_steps * n * (4 * k * c + 4 * k * k)
    timer = _Timer(torch)
    out = {}
    with prec_ctx(precision):
        seq = lstm_forward(params, x)
        lstm_backward(params, x, seq, dh)
        mode = "eager"
        try:  # each direction captured once into a CUDA graph: device time without host launch gaps
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            g_f, g_b = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_f, stream=side):
                seq_g = lstm_forward(params, x)
            with torch.cuda.graph(g_b, stream=side):
                lstm_backward(params, x, seq_g, dh)
            torch.cuda.synchronize()
            fwd_call, bwd_call = (lambda sp: g_f.replay()), (lambda sp: g_b.replay())
            mode = "cuda-graph"
        except Exception:  # noqa: BLE001 - fall back to eager launches
            fwd_call = lambda sp: lstm_forward(params, x)  # noqa: E731
            bwd_call = lambda sp: lstm_backward(params, x, seq, dh)  # noqa: E731
        fwd_mean, fwd_min = timer(fwd_call, iters, warmup=1)
        bwd_mean, bwd_min = timer(bwd_call, iters, warmup=1)
    peak, _, src = _peaks()
    out["fwd"] = {"ms": fwd_mean * 1e3, "tflops": flops_fwd / fwd_mean / 1e12}
    out["bwd_upd"] = {"ms": bwd_mean * 1e3, "tflops": 2 * flops_fwd / bwd_mean / 1e12}
    tot = 3 * flops_fwd / (fwd_mean + bwd_mean)
    out["all"] = {"tflops": tot / 1e12, "frac_of_peak": tot / (peak * 1e12), "gflop": 3 * flops_fwd / 1e9}
    out["config"] = {"T": t_steps, "N": n, "C": c, "K": k, "compute": precision, "storage": "fp32 h/s/gates",
                     "timing": mode}
    return out


def brgemm_suite(ms=(32, 64, 128, 256), batches=(1, 4, 16, 64), variants=("stride", "offset", "address"),
                 iters=10, max_bytes=1 << 30, square=True, precision="bf16"):
    """BASELINE config 5: BRGEMM shape sweep vs roofline (config 1 = stride, m=n=k=64, batch 16).

    Each point is ONE grouped launch of J independent output blocks C_j (the
    reference's single call is ~40-80 ns of ideal work), bf16
    inputs, fp32 C, beta = 0.  F = 2 m n k batch J; B = J (2 batch (mk + kn) + 4 mn).
    Reference storage contract (brgemm.py:1-24): a_i (k, m), b_i (n, k), c (n, m).
    precision "tf32": fp32 A/B in HBM (4-byte elements in B), TF32 tensor-core math —
    the reference's own fp32 storage (config 1 as written).
    """
    import torch

    from paper_1906_06440_b200 import _lib

    lib = _lib.load()
    peak, hbm, src = _peaks()
    timer = _Timer(torch)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    shapes = [(m, m, m) for m in ms] if square else [(m, n, k) for m in ms for n in ms for k in ms]
    rows = []
    tf32 = precision == "tf32"
    esz = 4 if tf32 else 2
    in_dt = _lib.BRK_F32 if tf32 else _lib.BRK_BF16
    comp = _lib.BRK_COMPUTE_TF32 if tf32 else _lib.BRK_COMPUTE_BF16
    for m, n, k in shapes:
        for batch in batches:
            per_job = esz * batch * (m * k + k * n) + 4 * m * n
            jobs = int(max(1, min(8 * sms, max_bytes // per_job)))
            a = torch.randn(jobs * batch * k * m, device="cuda")
            b = torch.randn(jobs * batch * n * k, device="cuda")
            if not tf32:
                a, b = a.bfloat16(), b.bfloat16()
            c = torch.empty(jobs * n * m, device="cuda")
            flops = 2.0 * m * n * k * batch * jobs
            t_roof = max(flops / (peak * 1e12), jobs * per_job / (hbm * 1e9))
            ji = torch.arange(jobs, device="cuda", dtype=torch.int64)
            bi = torch.arange(batch, device="cuda", dtype=torch.int64)
            a_off = ((ji[:, None] * batch + bi[None, :]) * (k * m)).reshape(-1).contiguous()
            b_off = ((ji[:, None] * batch + bi[None, :]) * (n * k)).reshape(-1).contiguous()
            c_ptr = (c.data_ptr() + ji * (n * m * 4)).contiguous()
            a_ptr = (a.data_ptr() + a_off * esz).contiguous()
            b_ptr = (b.data_ptr() + b_off * esz).contiguous()
            for var in variants:
                if var == "stride":
                    fn = lambda sp: _lib.check(lib.brk_brgemm_stride(  # noqa: E731
                        a.data_ptr(), b.data_ptr(), k * m, n * k, c.data_ptr(), jobs, batch * k * m, batch * n * k,
                        n * m, m, n, k, batch, m, k, m, 1.0, 0.0, in_dt, _lib.BRK_F32, comp, sp))
                elif var == "offset":
                    fn = lambda sp: _lib.check(lib.brk_brgemm_offs(  # noqa: E731
                        a.data_ptr(), b.data_ptr(), a_off.data_ptr(), b_off.data_ptr(), c_ptr.data_ptr(), jobs, m, n,
                        k, batch, m, k, m, 1.0, 0.0, in_dt, _lib.BRK_F32, comp, sp))
                else:  # address lists into two registered allocations (brk_brgemm_addr_views)
                    fn = lambda sp: _lib.check(lib.brk_brgemm_addr_views(  # noqa: E731
                        a_ptr.data_ptr(), b_ptr.data_ptr(), c_ptr.data_ptr(), a.data_ptr(), a.numel(), b.data_ptr(),
                        b.numel(), jobs, m, n, k, batch, m, k, m, 1.0, 0.0, in_dt, _lib.BRK_F32, comp, sp))
                mean, best = timer(fn, iters)
                rows.append({"m": m, "n": n, "k": k, "batch": batch, "variant": var, "jobs": jobs,
                             "us": mean * 1e6, "tflops": flops / mean / 1e12, "roof_frac": t_roof / mean,
                             "bound": "tensor" if flops / (peak * 1e12) >= jobs * per_job / (hbm * 1e9) else "hbm"})
            del a, b, c
    if tf32:
        peak = _tf32_peak(peak)
        for r in rows:  # roofline against the TF32 tensor peak (half the bf16 rate)
            f = 2.0 * r["m"] * r["n"] * r["k"] * r["batch"] * r["jobs"]
            b_ = r["jobs"] * (esz * r["batch"] * (r["m"] * r["k"] + r["k"] * r["n"]) + 4 * r["m"] * r["n"])
            t_roof = max(f / (peak * 1e12), b_ / (hbm * 1e9))
            r["roof_frac"] = t_roof / (r["us"] * 1e-6)
            r["bound"] = "tensor" if f / (peak * 1e12) >= b_ / (hbm * 1e9) else "hbm"
    return {"peak_tflops": peak, "hbm_gbs": hbm, "peak_source": src, "precision": precision, "points": rows}


def _tf32_peak(bf16_peak):
    """TF32 dense peak: the measured cuBLAS TF32 8192^3 number when profiles/ holds one
    (profiles/r02/dense_peak.json), else half the bf16 peak (tensor-core rate ratio)."""
    import json
    from pathlib import Path

    f = Path(__file__).resolve().parent.parent / "profiles" / "r02" / "dense_peak.json"
    try:
        d = json.loads(f.read_text())["dense_peak"]["8192x8192x8192"]
        return max(d["cublas_tf32_tflops"], d.get("engine_tf32_tflops", 0.0))
    except (OSError, KeyError, ValueError):
        return bf16_peak / 2


def split_gemm_baseline(m=64, n=64, k=64, batch=16, iters=10):
    """SURVEY 8(f)3 / reference tests/test_acceptance.py:268-292: the batch-reduce GEMM
    (the batch sum stays in TMEM, one store) against the split-GEMM formulation of the
    same work — one GEMM launch per batch entry accumulating C through memory
    (beta = 1).  BASELINE config 1 shape, 8 jobs per SM, bf16 -> fp32."""
    import torch

    from paper_1906_06440_b200 import _lib

    lib = _lib.load()
    timer = _Timer(torch)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    jobs = 8 * sms
    a = torch.randn(jobs * batch * k * m, device="cuda").bfloat16()
    b = torch.randn(jobs * batch * n * k, device="cuda").bfloat16()
    c = torch.empty(jobs * n * m, device="cuda")
    c2 = torch.empty_like(c)

    def stride(sp, base_a, base_b, nb, beta, out):
        _lib.check(lib.brk_brgemm_stride(base_a, base_b, k * m, n * k, out.data_ptr(), jobs, batch * k * m,
                                         batch * n * k, n * m, m, n, k, nb, m, k, m, 1.0, beta, _lib.BRK_BF16,
                                         _lib.BRK_F32, _lib.BRK_COMPUTE_BF16, sp))

    def brgemm(sp):
        stride(sp, a.data_ptr(), b.data_ptr(), batch, 0.0, c)

    def split(sp):
        for i in range(batch):
            stride(sp, a.data_ptr() + 2 * i * k * m, b.data_ptr() + 2 * i * n * k, 1, 0.0 if i == 0 else 1.0, c2)

    t_br, _ = timer(brgemm, iters)
    t_sp, _ = timer(split, iters)
    torch.cuda.synchronize()
    err = (c - c2).abs().max().item() / max(c.abs().max().item(), 1e-30)
    # HBM roofline of each arm: the BRGEMM reads every A/B block once and writes C once;
    # the split arm re-reads and re-writes C in every launch after the first
    _, hbm, _ = _peaks()
    ab = jobs * batch * 2 * (k * m + n * k)
    br_bytes = ab + jobs * 4 * n * m
    sp_bytes = ab + jobs * 4 * n * m * (2 * batch - 1)
    return {"shape": f"m=n=k={m} batch={batch} jobs={jobs}", "brgemm_us": t_br * 1e6, "split_gemm_us": t_sp * 1e6,
            "speedup": t_sp / t_br, "split_launches": batch, "max_rel_diff": err,
            "brgemm_hbm_roof_frac": br_bytes / (hbm * 1e9) / t_br,
            "split_hbm_roof_frac": sp_bytes / (hbm * 1e9) / t_sp,
            "roofline_speedup": sp_bytes / br_bytes,
            "note": "split arm = one beta=1 stride-BRGEMM launch per batch entry (batch 1), C through HBM; "
                    "roofline_speedup = the byte ratio, the speed-up an ideal kernel would show"}


def _dp_time(step, pg, iters, warmup=1):
    """Mean device time of ``step`` (CUDA events on the current stream), max over ranks."""
    import torch

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if pg is not None:
        import torch.distributed as dist
        dist.barrier(group=pg)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(iters):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) * 1e-3 / iters
    if pg is not None:
        import torch.distributed as dist
        t = torch.tensor([sec], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=pg)
        sec = float(t.item())
    return sec


def resnet_dp_suite(pg=None, n_global=256, iters=3):
    """ResNet-50's 53 convs as one data-parallel training step (train.ResNetConvs): global
    minibatch n_global split over the ranks (strong scaling), fwd + bwd-data + upd of every
    conv, per-layer dW all-reduce overlapping the backward, SGD.  Whole-job TFLOP/s."""
    from paper_1906_06440_b200.train import ResNetConvs

    import torch

    net = ResNetConvs(n_global=n_global, process_group=pg)
    sec = _dp_time(net.step, pg, iters)
    world = net.world
    flops = net.flops_per_step(local=False)
    peak, _, src = _peaks()
    out = {"n_global": n_global, "n_per_gpu": net.n_local, "gpus": world, "ms_per_step": sec * 1e3,
           "tflops": flops / sec / 1e12, "tflops_per_gpu": flops / sec / 1e12 / world,
           "frac_of_peak_per_gpu": flops / sec / 1e12 / world / peak, "gflop_per_step": flops / 1e9,
           "scaling": "strong", "convs": len(net.layers),
           "note": "53 convs (20 shapes x count), bf16, fwd + bwd-data (stem included) + upd, per-layer NCCL "
                   "all-reduce of dW on a comm stream in reverse order, SGD; device time, max over ranks"}
    del net
    torch.cuda.empty_cache()
    return out


def lstm_dp_suite(pg=None, n_per_gpu=168, iters=10):
    """LSTM cell C=K=1024, T=50 data parallel (train.LstmDP): N=168 sequences per rank (weak
    scaling), fwd + BPTT + weight update, dW/dR/db all-reduce overlapping dx, SGD."""
    from paper_1906_06440_b200.train import LstmDP

    import torch

    net = LstmDP(n_local=n_per_gpu, process_group=pg)
    # (a ~2 ms step: 3 warm-up steps settle the caching allocator after the ResNet suites, whose
    #  frees otherwise put cudaMalloc calls into the first timed steps)
    sec = _dp_time(net.step, pg, iters, warmup=3)
    world = net.world
    flops = net.flops_per_step() * world
    peak, _, src = _peaks()
    out = {"n_per_gpu": n_per_gpu, "n_global": n_per_gpu * world, "gpus": world, "ms_per_step": sec * 1e3,
           "tflops": flops / sec / 1e12, "tflops_per_gpu": flops / sec / 1e12 / world,
           "frac_of_peak_per_gpu": flops / sec / 1e12 / world / peak, "gflop_per_step": flops / 1e9,
           "scaling": "weak",
           "note": "T=50, C=K=1024, bf16 compute, fwd + BPTT + upd, dW/dR/db NCCL all-reduce overlapping dx, "
                   "SGD; device time, max over ranks"}
    del net
    torch.cuda.empty_cache()
    return out


def _plan(lib, pass_, geom):
    import ctypes
    out = (ctypes.c_int * 3)()
    lib.brk_conv_plan(pass_, *geom, out)
    return tuple(out)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "conv"
    if what == "conv":
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
        layers = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else None
        res = resnet_suite(n=n, layers=layers, verbose=True)
        for row in res["layers"]:
            cells = []
            for p in ("fwd", "bwd", "upd"):
                v = row.get(p)
                cells.append(f"{p} {v['us']:8.1f}us {v['tflops']:7.1f}TF {v['roof_frac']*100:5.1f}%roof"
                             if v else f"{p} {'n/a':>30}")
            print(f"L{row['id']:2d} x{row['count']} {row['path']:7s} {row.get('plan', '')}  " + " | ".join(cells))
        print(json.dumps(res["summary"], indent=1))
        (ROOT / "gpurun_out").mkdir(exist_ok=True)
        (ROOT / "gpurun_out" / f"resnet_n{n}.json").write_text(json.dumps(res, indent=1))
    elif what == "lstm":
        print(json.dumps(lstm_suite(), indent=1))
    elif what == "brgemm":
        res = brgemm_suite()
        for r in res["points"]:
            print(f"m=n=k={r['m']:3d} batch {r['batch']:2d} {r['variant']:7s} jobs {r['jobs']:5d}: {r['us']:9.1f} us "
                  f"{r['tflops']:7.1f} TF/s  {r['roof_frac'] * 100:5.1f}% of roofline ({r['bound']})")


def mlp_tf32_suite(layers=4, width=1024, batch=2048, iters=10):
    """BASELINE config 2 with the reference's fp32 storage and TF32 math (MlpTF32):
    whole step (one fused persistent launch, or 4L+1+L with BRK_MLP_FUSED=0) captured in a CUDA graph, L2 flushed
    between steps; TFLOP/s against the TF32 dense peak."""
    import torch

    from paper_1906_06440_b200.mlp import MlpTF32, flops_per_step

    m = MlpTF32(layers=layers, width=width, batch=batch, lr=1e-4, seed=0)
    g = torch.Generator(device="cuda").manual_seed(1)
    m.load_input(torch.rand(m.y[0].shape, generator=g, device="cuda") * 2 - 1,
                 torch.rand(m.dy.shape, generator=g, device="cuda") * 2 - 1)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        m.step(side.cuda_stream)
    side.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        m.step(side.cuda_stream)
    torch.cuda.synchronize()
    mean, best = _Timer(torch)(lambda sp: graph.replay(), iters)
    fl = flops_per_step(layers, batch, width, width)
    bf16_peak, _, _ = _peaks()
    peak = _tf32_peak(bf16_peak)
    return {"ms_per_step": mean * 1e3, "tflops": fl / mean / 1e12, "tf32_peak_tflops": peak,
            "frac_of_tf32_peak": fl / mean / 1e12 / peak, "launches_per_step": m.launches_per_step,
            "config": {"layers": layers, "C": width, "K": width, "N": batch, "storage": "fp32",
                       "compute": "tf32", "timing": "cuda-graph, L2 flushed"}}
