"""Benchmark: MLP 4 x FC(1024 -> 1024) + bias + ReLU, minibatch 2048 per GPU,
fwd / bwd-data / weight-update (+ bias grad + SGD) — BASELINE.json config 2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line (rank 0).  `value` is whole-job TFLOP/s (GEMM flops
3 * 2NCK per layer, the reference's flops_fc accounting, bench.py:112-113)
over device-timed steps with inputs resident in HBM; `e2e` repeats it through
the public MLP.train_step call with host->device copies of the step's input
and gradient from pinned memory and a device->host read of the result.
L2 is flushed (256 MiB write) between timed steps.  Multi-GPU: one process
per GPU (torchrun), data parallel, weak scaling (N=2048 per GPU), NCCL
all-reduce of dW/db per layer; time = max over ranks of device time.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port of the blocked FC BRGEMM loops, oracle/brk_oracle.py, all host
threads) on the same 4-layer step at the full size, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

LAYERS, WIDTH, BATCH = 4, 1024, 2048
METRIC = "TFLOP/s & % of B200 dense peak: ResNet-50 conv, LSTM cell, MLP fwd/bwd/upd"
UNIT = "TFLOP/s"
WORKLOAD = "mlp4x_fc1024_n2048_fwd_bwd_upd_bias_relu_sgd"


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def base_config(n_gpus):
    return {"workload": WORKLOAD, "layers": LAYERS, "C": WIDTH, "K": WIDTH, "N_per_gpu": BATCH,
            "global_batch": BATCH * n_gpus, "blocking": "b_n=b_c=b_k=64 (reference blocked FC layouts)",
            "bias": True, "activation": "relu", "sgd": "fused (upd epilogue / bias-grad kernel)",
            "parallelism": f"dp{n_gpus}", "l2": "flushed between timed steps (256 MiB write)"}


# ---------------------------------------------------------------------------
# clocks sampler
# ---------------------------------------------------------------------------
_REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[2], 16)
            except ValueError:
                continue
            for bit, name in _REASON_BITS.items():
                if bits & bit:
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [v for v in sm if v > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference arm (CPU)
# ---------------------------------------------------------------------------
def reference_step():
    """(step_fn, threads): one full MLP step of the benchmarked config (4 layers, C=K=1024,
    N=2048, bias + ReLU) with the reference's blocked FC BRGEMM algorithm on the host
    (oracle port of fc.py:99-163 over brgemm.py:260-293, float64 block accumulation, all
    host threads): forward through the 4 layers, then per layer from the top the
    backward-data, weight-update and bias-gradient passes (restated, oracle/brk_oracle.py).
    The reference is Python/NumPy and cannot travel to the GPU box, so its algorithm runs
    from the port; the SGD apply is elementwise and omitted (it has no GEMM flops)."""
    import numpy as np

    sys.path.insert(0, str(ROOT / "oracle"))
    import brk_oracle as orc

    threads = orc.cpu_threads()
    rng = np.random.default_rng([0, 202])
    b = 64
    blk_w = lambda w: w.reshape(WIDTH // b, b, WIDTH // b, b).transpose(0, 2, 3, 1).copy()  # noqa: E731
    blk_x = lambda x: x.reshape(BATCH // b, b, WIDTH // b, b).transpose(0, 2, 1, 3).copy()  # noqa: E731
    wbs = [blk_w((rng.uniform(-1, 1, (WIDTH, WIDTH)) / 32).astype(np.float32)) for _ in range(LAYERS)]
    biases = [rng.uniform(-0.1, 0.1, WIDTH).astype(np.float32) for _ in range(LAYERS)]
    xb = blk_x(rng.uniform(-1, 1, (BATCH, WIDTH)).astype(np.float32))
    dyb = blk_x(rng.uniform(-1, 1, (BATCH, WIDTH)).astype(np.float32))

    def step():
        ys = [xb]
        for wb, bias in zip(wbs, biases):
            ys.append(orc.fc_forward_blocked(wb, ys[-1], "relu", bias, workers=threads))
        d = dyb
        for l in range(LAYERS - 1, -1, -1):
            d, _, _ = orc.fc_backward_blocked(wbs[l], ys[l], ys[l + 1], d, "relu", workers=threads)

    return step, threads


REF_SAMPLE = (f"the full benchmarked MLP step ({LAYERS} x FC C=K={WIDTH}, N={BATCH}, bias+ReLU: fwd of every "
              f"layer, then bwd-data + weight-update + bias-grad of every layer) with the reference's blocked "
              f"BRGEMM algorithm (oracle port, float64 block accumulation)")


def run_reference(args, n_gpus, rank):
    if rank != 0:
        return
    step, threads = reference_step()
    flops = LAYERS * 3 * 2 * BATCH * WIDTH * WIDTH
    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    sec = statistics.fmean(times)
    value = flops / sec / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64-accumulate/f32-storage", "data": "synthetic",
            "config": base_config(n_gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{REF_SAMPLE}, {threads} threads, one step per timed step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_sample():
    """Bounded CPU sample for the GPU arm's cpu_baseline key (~10-30 s): whole reference steps."""
    step, threads = reference_step()
    reps, t_total = 0, 0.0
    while t_total < 10.0 and reps < 20:
        t0 = time.perf_counter()
        step()
        t_total += time.perf_counter() - t0
        reps += 1
    value = reps * LAYERS * 3 * 2 * BATCH * WIDTH * WIDTH / t_total / 1e12
    return {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{reps} x {REF_SAMPLE}, {t_total:.1f} s, {threads} threads"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def kernel_roofline(mlp, torch, peak_tflops):
    """Roofline block for the dominant kernel of the timed step: the lean
    persistent launch that runs the whole MLP step (brk_mlp_step,
    mlp_step_kernel in csrc/brk_mlp.cu).  Algorithmic FLOPs per launch = 12 *
    2NCK; time per launch from CUDA events around a graph of 10
    launches on the launching stream; traffic = ncu dram read + write bytes of
    one launch (profiles/r02/mlp_kernel_ncu.json).  The standalone per-pass kernels (the
    13-launch path) are timed the same way and reported alongside."""
    from paper_1906_06440_b200 import _lib
    from paper_1906_06440_b200.mlp import flops_per_step

    lib, n, c = mlp.lib, mlp.N, mlp.C
    B = 64
    stream = torch.cuda.Stream()

    def graph_time(fn, reps=10):
        with torch.cuda.stream(stream):
            fn(stream.cuda_stream)
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(reps):
                fn(stream.cuda_stream)
        with torch.cuda.stream(stream):
            for _ in range(3):
                g.replay()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(5):
                g.replay()
            e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / (5 * reps) * 1e-3

    step_flops = flops_per_step(mlp.L, n, c, c)
    t_step = graph_time(lambda s: mlp.fused_step(s)) if mlp.fused else None
    passes = {
        "fwd": lambda s: lib.brk_fc_fwd(mlp.y[0].data_ptr(), mlp.w[0].data_ptr(), mlp.bias[0].data_ptr(),
                                        mlp.y[1].data_ptr(), n, c, c, B, B, B, 1, _lib.BRK_BF16, s),
        "bwd": lambda s: lib.brk_fc_bwd_data(mlp.dz[2].data_ptr(), mlp.w[1].data_ptr(), mlp.y[1].data_ptr(),
                                             mlp.dz[1].data_ptr(), mlp.colsum[1].data_ptr(), n, c, c, B, B, B,
                                             _lib.BRK_BF16, s),
        "upd": lambda s: lib.brk_fc_upd(mlp.y[0].data_ptr(), mlp.dz[1].data_ptr(), mlp.dw[0].data_ptr(), None,
                                        0.0, mlp.colsum[1].data_ptr(), n // 32, mlp.db[0].data_ptr(), None, 0.0,
                                        mlp.upd_ws[0].data_ptr(), mlp.upd_ws[0].numel(),
                                        n, c, c, B, B, B, _lib.BRK_BF16, s),
    }
    per_pass = {k: graph_time(fn) * 1e6 for k, fn in passes.items()}
    traffic = None
    tf = ROOT / "profiles" / "r02" / "mlp_kernel_ncu.json"
    if tf.exists():
        try:
            for recs in json.loads(tf.read_text()).values():
                for r in recs:
                    if "mlp_step_kernel" in r["kernel"]:
                        rd = float(r["dram__bytes_read.sum"].split()[0])
                        wr = float(r["dram__bytes_write.sum"].split()[0])
                        traffic = (rd + wr) * 1e6  # ncu reports Mbyte
        except (ValueError, KeyError):
            traffic = None
    if t_step is None:  # data-parallel / unfused configuration: the per-pass engine kernel dominates
        t_step = statistics.fmean(per_pass.values()) * 1e-6
        step_flops = 2.0 * n * c * c
        kernel = "brk engine_kernel (one FC pass)"
    else:
        kernel = "brk mlp_step_kernel: the whole MLP step (12 GEMMs, 256x128 CTA-pair tiles) in one persistent launch"
    achieved = step_flops / t_step / 1e12
    return {"bound": "tensor", "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
            "frac": achieved / peak_tflops, "traffic": traffic, "kernel": kernel,
            "flops_per_launch": step_flops, "us_per_launch": t_step * 1e6,
            "standalone_pass_us": per_pass}


def other_workloads():
    """The metric's other two workloads on this GPU (informational; the headline
    is the MLP config): ResNet-50 conv fwd/bwd/upd at N=256 (reference weighted
    efficiency over the 53 convs) and the LSTM cell (T=50, N=168, C=K=1024)."""
    from tools.suites import brgemm_suite, lstm_suite, resnet_suite

    out = {}
    try:
        res = resnet_suite(n=256, iters=5, layers=list(range(1, 21)))
        out["resnet50_conv_n256"] = {
            "summary": res["summary"], "summary_engine_layers": res["summary_engine_layers"],
            "peak_tflops": res["peak_tflops"], "hbm_gbs": res["hbm_gbs"],
            "note": "all 53 convs (layers 1-20 weighted by count; layer-1 bwd-data excluded as in the reference "
                    "table), bf16 storage, L2 flushed between launches; layers 2-20 on the implicit-GEMM engine, "
                    "layer 1 (C=3 stem) as explicit im2col + the dense engine GEMM",
            "per_layer_us": {r["id"]: {p: round(r[p]["us"], 1) for p in ("fwd", "bwd", "upd") if r.get(p)}
                             for r in res["layers"]}}
    except Exception as exc:  # noqa: BLE001 - informational block must not kill the headline line
        out["resnet50_conv_n256"] = {"error": repr(exc)[:300]}
    try:  # the reference's fp32 storage with TF32 math, the engine layers (the C=3 stem stays bf16-only)
        res = resnet_suite(n=256, iters=3, layers=list(range(2, 21)), precision="tf32")
        out["resnet50_conv_n256_tf32"] = {
            "summary": res["summary"], "peak_tflops": res["peak_tflops"],
            "note": "layers 2-20 (52 convs weighted by count), fp32 storage, TF32 tcgen05 MMAs, L2 flushed; "
                    "roofline against the measured TF32 peak",
            "per_layer_us": {r["id"]: {p: round(r[p]["us"], 1) for p in ("fwd", "bwd", "upd") if r.get(p)}
                             for r in res["layers"]}}
    except Exception as exc:  # noqa: BLE001
        out["resnet50_conv_n256_tf32"] = {"error": repr(exc)[:300]}
    try:
        out["lstm_t50_n168_c1024"] = lstm_suite(iters=2)
    except Exception as exc:  # noqa: BLE001
        out["lstm_t50_n168_c1024"] = {"error": repr(exc)[:300]}
    try:  # configs 1 and 5: the reference-API BRGEMM (grouped launch of J independent C blocks)
        res = brgemm_suite(iters=5)
        pts = res["points"]
        c1 = [r for r in pts if r["m"] == 64 and r["batch"] == 16 and r["variant"] == "stride"][0]
        out["brgemm"] = {
            "config1_stride_16x64x64x64": {k: c1[k] for k in ("jobs", "us", "tflops", "roof_frac", "bound")},
            "sweep": [{k: r[k] for k in ("m", "batch", "variant", "jobs", "tflops", "roof_frac")} for r in pts],
            "note": "m=n=k in 32..256, batch 1..64, bf16 in / fp32 C, one grouped launch per point"}
        # config 1 as written: fp32 blocks in HBM, TF32 tensor-core math (north_star "TF32 inputs")
        r32 = brgemm_suite(ms=(64,), batches=(16,), iters=5, precision="tf32")
        out["brgemm"]["config1_stride_16x64x64x64_tf32"] = {
            r["variant"]: {k: r[k] for k in ("jobs", "us", "tflops", "roof_frac", "bound")} for r in r32["points"]}
        out["brgemm"]["tf32_peak_tflops"] = r32["peak_tflops"]
        # config 5: independent M, N, K in {32, 64, 128, 256} (batch 16), every variant
        grid = brgemm_suite(batches=(16,), iters=3, square=False)["points"]
        out["brgemm"]["grid_mnk_batch16"] = {
            "points": [[r["m"], r["n"], r["k"], r["variant"], round(r["tflops"], 1), round(r["roof_frac"], 3)]
                       for r in grid],
            "columns": ["m", "n", "k", "variant", "tflops", "roof_frac"],
            "median_roof_frac": {v: statistics.median(r["roof_frac"] for r in grid if r["variant"] == v)
                                 for v in ("stride", "offset", "address")}}
    except Exception as exc:  # noqa: BLE001
        out["brgemm"] = {"error": repr(exc)[:300]}
    try:  # the headline config with the reference's fp32 storage, TF32 tensor-core math
        from tools.suites import mlp_tf32_suite
        out["mlp4x1024_n2048_tf32"] = mlp_tf32_suite()
    except Exception as exc:  # noqa: BLE001
        out["mlp4x1024_n2048_tf32"] = {"error": repr(exc)[:300]}
    try:  # TMEM-resident batch reduction vs split GEMMs accumulating through memory
        from tools.suites import split_gemm_baseline
        out["brgemm_vs_split_gemm"] = split_gemm_baseline(iters=5)
    except Exception as exc:  # noqa: BLE001
        out["brgemm_vs_split_gemm"] = {"error": repr(exc)[:300]}
    return out


def dp_workloads(pg):
    """The conv and LSTM workloads as data-parallel training steps at this world size
    (train.py): ResNet-50's 53 convs at global minibatch 256 (strong scaling) and the
    LSTM cell at N=168 per GPU (weak scaling); whole-job TFLOP/s, max over ranks."""
    from tools.suites import lstm_dp_suite, resnet_dp_suite

    out = {}
    for name, fn in (("resnet50_convs_dp_n256", resnet_dp_suite), ("lstm_dp_n168_per_gpu", lstm_dp_suite)):
        try:
            out[name] = fn(pg)
        except Exception as exc:  # noqa: BLE001 - informational block must not kill the headline line
            out[name] = {"error": repr(exc)[:300]}
    return out


def run_gpu(args, n_gpus, rank, local_rank, pg):
    import torch

    from paper_1906_06440_b200 import _lib
    from paper_1906_06440_b200.mlp import MLP, flops_per_step

    torch.cuda.set_device(local_rank)
    pk, pk_kind = peaks()
    mlp = MLP(layers=LAYERS, width=WIDTH, batch=BATCH, lr=1e-4, seed=0, process_group=pg)  # data: seed 100+rank
    g = torch.Generator(device="cpu").manual_seed(100 + rank)
    blk = lambda t: t.reshape(BATCH // 64, 64, WIDTH // 64, 64).permute(0, 2, 1, 3).contiguous()  # noqa: E731
    x_host = blk((torch.rand(BATCH, WIDTH, generator=g) * 2 - 1).bfloat16()).pin_memory()
    dy_host = blk(((torch.rand(BATCH, WIDTH, generator=g) * 2 - 1) * 1e-2).bfloat16()).pin_memory()
    mlp.load_input(x_host.cuda(), dy_host.cuda())
    torch.cuda.synchronize()
    single = pg is None
    if single:
        mlp.capture()
        run = mlp.replay
    else:
        run = mlp.step
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    flops = flops_per_step(LAYERS, BATCH, WIDTH, WIDTH)
    stream = torch.cuda.current_stream()

    def barrier():
        if pg is not None:
            import torch.distributed as dist
            dist.barrier(group=pg)

    def timed(step_fn, steps):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        barrier()
        torch.cuda.synchronize()
        for i in range(steps):
            flush.fill_(float(i))                     # L2 flush, outside the timed events
            evs[i][0].record(stream)
            step_fn()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        barrier()
        return sum(a.elapsed_time(b) for a, b in evs) * 1e-3 / steps

    def max_over_ranks(v):
        if pg is None:
            return v
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=pg)
        return float(t.item())

    with ClockSampler(local_rank) as clk:
        # clock ramp + warm-up (at least W steps, and ~1 s of device work)
        t_end = time.time() + 1.0
        w = 0
        while w < args.warmup or time.time() < t_end:
            run()
            w += 1
        torch.cuda.synchronize()
        sec = max_over_ranks(timed(run, args.steps))
        # end-to-end through the public API (MLP.train): every step copies its input and
        # output gradient from pinned host memory (overlapping the previous step's compute)
        # and reads its result back; device time of the whole pipelined sequence / steps
        outs = [torch.empty(WIDTH, dtype=torch.float32, pin_memory=True) for _ in range(args.steps)]
        xs, dys = [x_host] * args.steps, [dy_host] * args.steps
        mlp.train(xs[:3], dys[:3], outs[:3])  # warm the copy stream and staging buffers
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        mlp.train(xs, dys, outs)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_sec = max_over_ranks(e0.elapsed_time(e1) * 1e-3 / args.steps)
    clocks = clk.summary()
    launches = mlp.launches_per_step
    value = n_gpus * flops / sec / 1e12
    e2e_value = n_gpus * flops / e2e_sec / 1e12
    suites = os.environ.get("BRK_BENCH_SUITES", "1") != "0"
    dp = dp_workloads(pg) if suites else None  # every rank takes part (collectives)
    if rank != 0:
        return
    workloads = None
    if n_gpus == 1 and suites:
        workloads = other_workloads()
    if dp is not None:
        workloads = dict(workloads or {}, **dp)
    roof = kernel_roofline(mlp, torch, pk["bf16_tflops"])
    roof["peak_source"] = f"{pk_kind} bf16 dense (burst, kernel timed alone)"
    cpu = cpu_baseline_sample()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform, seeded; random-init weights)",
        "config": base_config(n_gpus),
        "pct_of_peak": value / n_gpus / pk["bf16_tflops_sustained"],
        "peak_note": f"{pk_kind} bf16 sustained {pk['bf16_tflops_sustained']} TFLOP/s per GPU",
        "flops_per_step_per_gpu": flops,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * BATCH * WIDTH * 2,
                "d2h_bytes_per_step": WIDTH * 4, "ms_per_step": e2e_sec * 1e3,
                "api": "MLP.train: pinned-host H2D of x and dy every step on a copy stream overlapping the "
                       "previous step, graph-replayed step, D2H of db; device time of the whole sequence"},
        "gpu_launches": launches * args.steps,
        "launches_per_step": launches,
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "lib_launch_counter": _lib.launch_count(),
        "workloads": workloads,
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args) -> int:
    """Re-launch this script under torch.distributed.run with one rank per GPU."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}", file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()),
           "--gpus", str(args.gpus), "--steps", str(args.steps), "--warmup", str(args.warmup)]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["brk", "reference"], default="brk")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, world if world > 1 else args.gpus, rank)
        return
    if world == 1 and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus N without a launcher: start N ranks ourselves (one process per GPU),
        # never scale a one-process number
        sys.exit(spawn_ranks(args))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    n_gpus = world
    pg = None
    if world > 1 or os.environ.get("BRK_FORCE_DP") == "1":  # torchrun: NCCL data parallel
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        pg = dist.group.WORLD
    try:
        run_gpu(args, n_gpus, rank, local_rank, pg)
    finally:
        if pg is not None:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
