"""The GPU benchmark CLI (reference bench.py subcommands, CSV rows) runs end to end,
mirroring the reference's own CLI acceptance test (test_acceptance.py:295-326):
all 20 conv layers verified at N=2, the other subcommands with --verify, --dump
writing the reference's binary tensor files, --include-reformat timing the
device layout kernels, and every timed call captured in a CUDA graph."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1906_06440_b200.bench import CSV_HEADER, BenchConfig, run_suite  # noqa: E402
from paper_1906_06440_b200.tensor import load_tensor  # noqa: E402


def test_cli_conv_all_layers_verified(tmp_path, capsys):
    out = tmp_path / "conv.csv"
    assert run_suite(BenchConfig("conv", layers="1-20", minibatch=2, iters=3, verify=True, csv=str(out))) == 0
    lines = out.read_text().strip().splitlines()
    assert lines[0] == CSV_HEADER
    rows = [r.split(",") for r in lines[1:]]
    assert len(rows) == 20
    for f in rows:
        assert f[0] == "conv" and f[2] == "2" and f[8] == "true"
        assert float(f[5]) > 0 and float(f[6]) > 0 and float(f[7]) > 0
        assert float(f[11]) <= 1.2, f"roofline fraction above 1.2: {f}"
    err = capsys.readouterr().err
    assert "timed eagerly" not in err, err


def test_cli_other_workloads_verify_dump_and_baseline(tmp_path, capsys):
    d = tmp_path / "dump"
    assert run_suite(BenchConfig("conv", layers="13", minibatch=2, iters=2, dump=str(d))) == 0
    for name in ("input", "weights", "output"):
        t = load_tensor(d / f"conv_13_{name}.bin")
        assert t.dtype == np.float32 and t.ndim == 4
    assert run_suite(BenchConfig("fc", minibatch=128, c=256, k=256, iters=2, verify=True, dump=str(d))) == 0
    assert load_tensor(d / "fc_output.bin").shape == (128, 256)
    assert run_suite(BenchConfig("lstm", minibatch=8, c=128, k=128, t_steps=3, iters=1, verify=True,
                                 dump=str(d))) == 0
    assert load_tensor(d / "lstm_hidden.bin").shape == (3, 8, 128)
    assert run_suite(BenchConfig("brgemm", iters=3, baseline=True)) == 0
    captured = capsys.readouterr()
    text = captured.out
    assert "brgemm_baseline,0,1," in text and "fc,0,128," in text and "lstm,0,8," in text
    assert "timed eagerly" not in captured.err, captured.err


def test_cli_include_reformat_costs_time(capsys):
    base = BenchConfig("conv", layers="2", minibatch=8, iters=5)
    assert run_suite(base) == 0
    plain = capsys.readouterr().out.strip().splitlines()[1].split(",")
    base.include_reformat = True
    assert run_suite(base) == 0
    ref = capsys.readouterr().out.strip().splitlines()[1].split(",")
    # the dense -> blocked transforms of input and weights plus the output unblock add time
    assert float(ref[5]) > float(plain[5])
