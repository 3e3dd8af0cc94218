"""Measurement API and GPU benchmark CLI (reference ``brkernels.bench``, bench.py:50-560).

Keeps the reference's FLOP accounting, ResNet-50 layer table, weighted
efficiency and CLI (subcommands ``conv`` / ``lstm`` / ``fc`` / ``brgemm``, the
same flags, the same CSV columns first) so GPU results compare row for row
with the reference's CPU table; the CSV adds ``dtype,gpus,roof_frac``.
Timing is on the device (CUDA events around each call, after warm-up).

    python -m paper_1906_06440_b200.bench conv --layers 1-20 --minibatch 28 --csv conv.csv
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .brgemm import BrgemmSpec
from .cnn import ConvSpec

CSV_HEADER = "workload,id,N,workers,flops,seconds_mean,seconds_min,gflops,verified,dtype,gpus,roof_frac"
VERIFY_TOL = {"bf16": 1e-2, "tf32": 1e-3}  # scale-relative (the reference's 1e-5 is its fp64-accumulate path)
DEFAULT_ITERS = 50

# (id, C, K, H, W, R, S, stride, count): the 20 distinct ResNet-50 convolutions, 53 in all
_RESNET50_ROWS = (
    (1, 3, 64, 224, 224, 7, 7, 2, 1), (2, 64, 256, 56, 56, 1, 1, 1, 4), (3, 64, 64, 56, 56, 1, 1, 1, 1),
    (4, 64, 64, 56, 56, 3, 3, 1, 3), (5, 256, 64, 56, 56, 1, 1, 1, 2), (6, 256, 512, 56, 56, 1, 1, 2, 1),
    (7, 256, 128, 56, 56, 1, 1, 2, 1), (8, 128, 128, 28, 28, 3, 3, 1, 4), (9, 128, 512, 28, 28, 1, 1, 1, 4),
    (10, 512, 128, 28, 28, 1, 1, 1, 3), (11, 512, 1024, 28, 28, 1, 1, 2, 1), (12, 512, 256, 28, 28, 1, 1, 2, 1),
    (13, 256, 256, 14, 14, 3, 3, 1, 6), (14, 256, 1024, 14, 14, 1, 1, 1, 6), (15, 1024, 256, 14, 14, 1, 1, 1, 5),
    (16, 1024, 2048, 14, 14, 1, 1, 2, 1), (17, 1024, 512, 14, 14, 1, 1, 2, 1), (18, 512, 512, 7, 7, 3, 3, 1, 3),
    (19, 512, 2048, 7, 7, 1, 1, 1, 3), (20, 2048, 512, 7, 7, 1, 1, 1, 2),
)


@dataclass(frozen=True)
class LayerRecord:
    """One ResNet-50 layer row: the conv problem and how often it occurs (bench.py:82-88)."""

    layer_id: int
    spec: ConvSpec
    count: int


def resnet50_table(minibatch: int = 1) -> list[LayerRecord]:
    """The 20 distinct ResNet-50 convolutions at a mini-batch (bench.py:91-97)."""
    return [LayerRecord(lid, ConvSpec(n=minibatch, c=c, k=k, h=h, w=w, r=r, s=s, stride=st), cnt)
            for lid, c, k, h, w, r, s, st, cnt in _RESNET50_ROWS]


def flops_conv(spec: ConvSpec, n: int) -> int:
    """2 N K C R S P Q (bench.py:100-102)."""
    return 2 * n * spec.k * spec.c * spec.r * spec.s * spec.out_h * spec.out_w


def flops_lstm_fwd(t_steps: int, n: int, c: int, k: int) -> int:
    """GEMM flops of the LSTM forward pass, 2 T N (4KC + 4KK) (bench.py:105-110)."""
    return 2 * t_steps * n * (4 * k * c + 4 * k * k)


def flops_fc(n: int, c: int, k: int) -> int:
    return 2 * n * c * k


def flops_brgemm(spec: BrgemmSpec) -> int:
    return 2 * spec.m * spec.n * spec.k * spec.batch


@dataclass
class BenchResult:
    """Counted flops and measured seconds of one workload (bench.py:121-140)."""

    flops: int
    seconds_mean: float
    seconds_min: float
    iterations: int
    workers: int
    verified: bool | None = None

    def __post_init__(self):
        if self.seconds_mean <= 0 or self.seconds_min <= 0:
            raise ValueError("measured time must be > 0")

    @property
    def rate(self) -> float:
        return self.flops / self.seconds_mean


def weighted_efficiency(results: list[tuple[BenchResult, int]], peak_flops: float) -> float:
    """(sum n_i F_i) / (sum n_i t_i) / peak over a layer multiset (bench.py:142-152)."""
    if not results:
        raise ValueError("weighted_efficiency needs at least one result")
    if peak_flops <= 0:
        raise ValueError(f"peak must be > 0, got {peak_flops}")
    num = sum(n_i * r.flops for r, n_i in results)
    den = sum(n_i * r.seconds_mean for r, n_i in results)
    if den <= 0:
        raise ValueError("aggregate time must be > 0")
    return num / den / peak_flops


def parse_layers(text: str, low: int = 1, high: int = 20) -> list[int]:
    """'1-20', '13' or '1,4,8-10' -> sorted layer ids (bench.py:224-238)."""
    ids: set[int] = set()
    for part in (p.strip() for p in text.split(",")):
        if "-" in part:
            a, b = part.split("-", 1)
            ids.update(range(int(a), int(b) + 1))
        elif part:
            ids.add(int(part))
    if not ids or any(not low <= i <= high for i in ids):
        raise ValueError(f"layer ids must be in {low}..{high}, got {sorted(ids)}")
    return sorted(ids)


@dataclass
class BenchConfig:
    """Parsed CLI options (bench.py:198-221)."""

    workload: str
    layers: str = "1-20"
    minibatch: int = 28
    workers: int = 1
    iters: int = DEFAULT_ITERS
    verify: bool = False
    peak_gflops: float | None = None
    csv: str | None = None
    dump: str | None = None
    include_reformat: bool = False
    seed: int = 0
    c: int = 256
    k: int = 256
    t_steps: int = 50
    activation: str = "relu"
    m: int = 64
    n: int = 6
    k_dim: int = 64
    batch: int = 16
    baseline: bool = False


def _peaks():
    root = Path(__file__).resolve().parents[1]
    try:
        d = json.loads((root / "MEASURED_PEAKS.json").read_text())
        return float(d["bf16_tflops"]), float(d["hbm_gbs"])
    except (OSError, ValueError, KeyError):  # the profiling guide's B200 fallbacks
        return 1590.0, 6650.0


def _time(fn, iters: int) -> tuple[float, float]:
    """Device seconds per call (mean, min).  The call is captured once in a CUDA graph and
    the graph replayed, so host-side argument handling of small problems does not show up
    as device idle time; calls that cannot be captured are timed eagerly."""
    import torch
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    run = fn
    try:
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                fn()
        torch.cuda.current_stream().wait_stream(side)
        graph.replay()
        torch.cuda.synchronize()
        run = graph.replay
    except Exception as exc:  # noqa: BLE001 - uncapturable call: eager timing, said out loud
        torch.cuda.synchronize()
        _log(f"note: call not capturable in a CUDA graph ({type(exc).__name__}); timed eagerly "
             f"(host-side work included)")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in evs:
        a.record()
        run()
        b.record()
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) * 1e-3 for a, b in evs]
    return statistics.fmean(ts), min(ts)


def _row(workload, lid, n, cfg, flops, res, verified, bytes_=0.0) -> str:
    peak, hbm = _peaks()
    if res is not None:
        mean, tmin = f"{res.seconds_mean:.9e}", f"{res.seconds_min:.9e}"
        gflops = f"{flops / res.seconds_mean / 1e9:.3f}"
        roof = f"{max(flops / (peak * 1e12), bytes_ / (hbm * 1e9)) / res.seconds_mean:.4f}"
    else:
        mean = tmin = gflops = roof = "nan"
    vtext = "" if verified is None else ("true" if verified else "false")
    return f"{workload},{lid},{n},{cfg.workers},{flops},{mean},{tmin},{gflops},{vtext},bf16,1,{roof}"


def _log(msg: str) -> None:
    print(msg, file=sys.stderr)


def _verify(got, ref, name) -> bool:
    err = float(np.max(np.abs(np.asarray(got, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-30))
    ok = err <= VERIFY_TOL["bf16"]
    _log(f"{name} verify={'ok' if ok else 'FAIL'} scale_rel_err={err:.2e}")
    return ok


def _maybe_dump(cfg: "BenchConfig", name: str, tensor) -> None:
    """--dump DIR: the reference's binary dump of a workload's tensors (reference bench.py:267-271)."""
    if cfg.dump:
        from .tensor import dump_tensor
        d = Path(cfg.dump)
        d.mkdir(parents=True, exist_ok=True)
        dump_tensor(tensor, d / f"{name}.bin")


def _oracle():
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root / "oracle"))  # test infrastructure: only for --verify
    import brk_oracle
    return brk_oracle


def _run_conv(cfg: BenchConfig, rows: list[str]) -> int:
    import torch

    from .cnn import conv2d_forward
    from .tensor import block_conv_tensors, unblock_conv_output
    failures, timed = 0, []
    records = {r.layer_id: r for r in resnet50_table(cfg.minibatch)}
    for lid in parse_layers(cfg.layers):
        rec = records[lid]
        spec = rec.spec
        rng = np.random.default_rng([cfg.seed, lid])
        i_d = rng.uniform(-1, 1, (spec.n, spec.c, spec.h, spec.w)).astype(np.float32)
        w_d = rng.uniform(-1, 1, (spec.k, spec.c, spec.r, spec.s)).astype(np.float32)
        inp, wgt = block_conv_tensors(i_d, w_d, spec.b_c, spec.b_k)
        inp, wgt = inp.to("cuda", torch.bfloat16), wgt.to("cuda", torch.bfloat16)
        flops = flops_conv(spec, spec.n)
        verified = None
        if cfg.verify or cfg.dump:
            got = unblock_conv_output(conv2d_forward(spec, inp, wgt).to("cpu"))
            if cfg.verify:
                ref = _oracle().conv2d_forward_reference(i_d, w_d, stride=spec.stride, pad_h=spec.pad_h,
                                                         pad_w=spec.pad_w)
                verified = _verify(got, ref, f"conv id={lid}")
                failures += 0 if verified else 1
            _maybe_dump(cfg, f"conv_{lid:02d}_input", i_d)
            _maybe_dump(cfg, f"conv_{lid:02d}_weights", w_d)
            _maybe_dump(cfg, f"conv_{lid:02d}_output", got)
        res = None
        if cfg.iters > 0:
            if cfg.include_reformat:
                # the paper's reformatting cost on the device: dense fp32 NCHW / KCRS
                # -> blocked bf16 (layout kernel, conversion fused), the conv, blocked -> dense fp32 output
                i_dev, w_dev = torch.from_numpy(i_d).cuda(), torch.from_numpy(w_d).cuda()

                def step():
                    xi, wi = block_conv_tensors(i_dev, w_dev, spec.b_c, spec.b_k, dtype=torch.bfloat16)
                    unblock_conv_output(conv2d_forward(spec, xi, wi))
            else:
                def step():
                    conv2d_forward(spec, inp, wgt)
            mean, tmin = _time(step, cfg.iters)
            res = BenchResult(flops, mean, tmin, cfg.iters, cfg.workers, verified)
            timed.append((res, rec.count))
        # algorithmic bytes: a 1x1 strided conv reads only the sampled input pixels
        in_px = spec.out_h * spec.out_w if (spec.r == 1 and spec.s == 1 and spec.stride > 1) else spec.h * spec.w
        nbytes = 2.0 * (spec.n * spec.c * in_px + spec.k * spec.c * spec.r * spec.s +
                        spec.n * spec.k * spec.out_h * spec.out_w)
        rows.append(_row("conv", lid, spec.n, cfg, flops, res, verified, nbytes))
    if timed:
        peak = cfg.peak_gflops * 1e9 if cfg.peak_gflops else _peaks()[0] * 1e12
        _log(f"weighted efficiency {weighted_efficiency(timed, peak):.4f} of {peak / 1e12:.0f} TFLOP/s")
    return failures


def _run_lstm(cfg: BenchConfig, rows: list[str]) -> int:
    import torch

    from . import precision
    from .lstm import LstmCellWeights, LstmParams, lstm_forward
    rng = np.random.default_rng([cfg.seed, 101])  # reference bench.py:331-334
    t_steps, n, c, k = cfg.t_steps, cfg.minibatch, cfg.c, cfg.k
    weights = LstmCellWeights.random(rng, c, k)
    x_h = rng.uniform(-1, 1, (t_steps, n, c)).astype(np.float32)
    params = LstmParams.from_dense(weights, t_steps, n)
    x = torch.from_numpy(x_h).cuda()
    flops = flops_lstm_fwd(t_steps, n, c, k)
    failures, verified = 0, None
    with precision("bf16"):
        if cfg.verify or cfg.dump:
            seq = lstm_forward(params, x_h)
            if cfg.verify:
                orc = _oracle()
                g = ("i", "c", "f", "o")
                ref = orc.lstm_forward_reference({q: getattr(weights, f"w_{q}") for q in g},
                                                 {q: getattr(weights, f"r_{q}") for q in g},
                                                 {q: getattr(weights, f"bias_{q}") for q in g}, x_h)
                verified = _verify(seq.h, ref["h"], "lstm h") and _verify(seq.s, ref["s"], "lstm s")
                failures += 0 if verified else 1
            _maybe_dump(cfg, "lstm_input", x_h)
            _maybe_dump(cfg, "lstm_hidden", seq.h)
            _maybe_dump(cfg, "lstm_state", seq.s)
        res = None
        if cfg.iters > 0:
            if cfg.include_reformat:  # re-block the weights every call (reference bench.py:350-353)
                def step():
                    lstm_forward(LstmParams.from_dense(weights, t_steps, n), x)
            else:
                def step():
                    lstm_forward(params, x)
            mean, tmin = _time(step, cfg.iters)
            res = BenchResult(flops, mean, tmin, cfg.iters, cfg.workers, verified)
    rows.append(_row("lstm", 0, n, cfg, flops, res, verified))
    return failures


def _run_fc(cfg: BenchConfig, rows: list[str]) -> int:
    import torch

    from .fc import Activation, FcParams, fc_forward
    from .tensor import block_fc_activation, unblock_fc_activation
    rng = np.random.default_rng([cfg.seed, 202])  # reference bench.py:374-378
    n, c, k = cfg.minibatch, cfg.c, cfg.k
    act = Activation(cfg.activation)
    w = rng.uniform(-1, 1, (k, c)).astype(np.float32)
    x_d = rng.uniform(-1, 1, (n, c)).astype(np.float32)
    params = FcParams.from_dense(w, n, activation=act)
    params.w = params.w.to("cuda", torch.bfloat16)
    x = block_fc_activation(x_d, params.b_n, params.b_c).to("cuda", torch.bfloat16)
    flops = flops_fc(n, c, k)
    failures, verified = 0, None
    if cfg.verify or cfg.dump:
        y = unblock_fc_activation(fc_forward(params, x).to("cpu"))
        if cfg.verify:
            ref = _oracle().fc_forward_reference(w, x_d.T, act.value).T
            verified = _verify(y, ref, "fc")
            failures += 0 if verified else 1
        _maybe_dump(cfg, "fc_input", x_d)
        _maybe_dump(cfg, "fc_weights", w)
        _maybe_dump(cfg, "fc_output", y)
    res = None
    if cfg.iters > 0:
        if cfg.include_reformat:  # dense fp32 on device -> blocked bf16 (layout kernel) every call
            w_dev, x_dev = torch.from_numpy(w).cuda(), torch.from_numpy(x_d).cuda()
            from .tensor import block_weight_2d

            def step():
                p = FcParams(w=block_weight_2d(w_dev, params.b_c, params.b_k, dtype=torch.bfloat16), n=n, c=c, k=k,
                             b_n=params.b_n, b_c=params.b_c, b_k=params.b_k, activation=act)
                unblock_fc_activation(fc_forward(p, block_fc_activation(x_dev, p.b_n, p.b_c, dtype=torch.bfloat16)))
        else:
            def step():
                fc_forward(params, x)
        mean, tmin = _time(step, cfg.iters)
        res = BenchResult(flops, mean, tmin, cfg.iters, cfg.workers, verified)
    rows.append(_row("fc", 0, n, cfg, flops, res, verified, 2.0 * (n * c + k * c + n * k)))
    return failures


def _run_brgemm(cfg: BenchConfig, rows: list[str]) -> int:
    import torch

    from .brgemm import batched_gemm, brgemm_strided
    m, n, k, batch = cfg.m, cfg.n, cfg.k_dim, cfg.batch
    spec = BrgemmSpec(m=m, n=n, k=k, batch=batch, beta=0.0)
    a = torch.randn(batch, k, m, device="cuda").bfloat16()
    b = torch.randn(batch, n, k, device="cuda").bfloat16()
    c = torch.zeros(n, m, device="cuda")
    flops = flops_brgemm(spec)
    mean, tmin = _time(lambda: brgemm_strided(a, b, k * m, n * k, c, spec), max(cfg.iters, 1))
    rows.append(_row("brgemm", 0, 1, cfg, flops, BenchResult(flops, mean, tmin, cfg.iters, 1), None,
                     2.0 * batch * (k * m + n * k) + 4.0 * n * m))
    if cfg.baseline:  # batched GEMM: one output per pair, no reduction (brgemm.py:340-353)
        from . import _lib
        from ._device import ptr_table, stream_ptr
        cs = torch.zeros(batch, n, m, device="cuda")
        batched_gemm(list(a), list(b), list(cs), spec)  # the public call once (checks, warm-up)
        # the same launch batched_gemm issues, with its address tables built once outside the
        # timed call so the graph capture sees only the kernel
        ta = ptr_table([t.data_ptr() for t in a])
        tb = ptr_table([t.data_ptr() for t in b])
        tc = ptr_table([t.data_ptr() for t in cs])
        lib = _lib.load()

        def base():
            _lib.check(lib.brk_brgemm_addr(ta.data_ptr(), tb.data_ptr(), tc.data_ptr(), batch, m, n, k, 1, m, k, m,
                                           1.0, 0.0, _lib.BRK_BF16, _lib.BRK_F32, _lib.BRK_COMPUTE_BF16,
                                           stream_ptr()))
        mean, tmin = _time(base, max(cfg.iters, 1))
        rows.append(_row("brgemm_baseline", 0, 1, cfg, flops, BenchResult(flops, mean, tmin, cfg.iters, 1), None,
                         2.0 * batch * (k * m + n * k) + 4.0 * batch * n * m))
    return 0


_RUNNERS = {"conv": _run_conv, "lstm": _run_lstm, "fc": _run_fc, "brgemm": _run_brgemm}


def run_suite(cfg: BenchConfig) -> int:
    """Run one workload family, print (and optionally write) the CSV; 1 if a verify failed."""
    rows: list[str] = []
    failures = _RUNNERS[cfg.workload](cfg, rows)
    text = "\n".join([CSV_HEADER] + rows)
    print(text)
    if cfg.csv:
        Path(cfg.csv).write_text(text + "\n")
    return 1 if failures else 0


def _build_parser() -> argparse.ArgumentParser:
    common = argparse.ArgumentParser(add_help=False)
    common.add_argument("--minibatch", type=int, help="mini-batch size N")
    common.add_argument("--workers", type=int, default=1)
    common.add_argument("--iters", type=int, default=DEFAULT_ITERS, help="timed iterations (0 = verify only)")
    common.add_argument("--verify", action="store_true", help="check against the fp64 oracle before timing")
    common.add_argument("--peak-gflops", type=float, default=None, help="peak GFLOP/s for efficiency")
    common.add_argument("--csv", type=str, default=None, help="CSV output path")
    common.add_argument("--dump", type=str, default=None, help="directory for binary tensor dumps")
    common.add_argument("--include-reformat", action="store_true",
                        help="time the dense -> blocked layout transforms (device kernel) with each call")
    common.add_argument("--seed", type=int, default=0)
    parser = argparse.ArgumentParser(prog="bench", description="Batch-reduce GEMM kernel benchmarks (B200)")
    sub = parser.add_subparsers(dest="workload", required=True)
    p = sub.add_parser("conv", parents=[common], help="ResNet-50 layer table")
    p.add_argument("--layers", type=str, default="1-20")
    p.set_defaults(minibatch_default=28)
    p = sub.add_parser("lstm", parents=[common], help="LSTM forward")
    p.add_argument("--C", dest="c", type=int, default=256)
    p.add_argument("--K", dest="k", type=int, default=256)
    p.add_argument("--T", dest="t_steps", type=int, default=50)
    p.set_defaults(minibatch_default=168)
    p = sub.add_parser("fc", parents=[common], help="fully connected forward layer")
    p.add_argument("--C", dest="c", type=int, default=512)
    p.add_argument("--K", dest="k", type=int, default=512)
    p.add_argument("--activation", type=str, default="relu", choices=["identity", "relu", "sigmoid"])
    p.set_defaults(minibatch_default=1344)
    p = sub.add_parser("brgemm", parents=[common], help="raw batch-reduce GEMM")
    p.add_argument("--m", type=int, default=64)
    p.add_argument("--n", type=int, default=6)
    p.add_argument("--k", dest="k_dim", type=int, default=64)
    p.add_argument("--batch", type=int, default=16)
    p.add_argument("--baseline", action="store_true", help="also run the batched-GEMM baseline")
    p.set_defaults(minibatch_default=1)
    return parser


def main(argv=None) -> None:
    args = _build_parser().parse_args(argv)
    kwargs = dict(vars(args))
    mb = kwargs.pop("minibatch_default", 1)
    if kwargs.get("minibatch") is None:
        kwargs["minibatch"] = mb
    try:
        code = run_suite(BenchConfig(**kwargs))
    except ValueError as exc:
        _log(f"error: {exc}")
        code = 2
    sys.exit(code)


if __name__ == "__main__":
    main()
