"""The GPU benchmark CLI (reference bench.py subcommands, CSV rows) runs end to end."""

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1906_06440_b200.bench import BenchConfig, run_suite  # noqa: E402


def test_cli_conv_verify_and_brgemm_rows(capsys, tmp_path):
    out = tmp_path / "conv.csv"
    assert run_suite(BenchConfig("conv", layers="1,13", minibatch=2, iters=2, verify=True, csv=str(out))) == 0
    rows = out.read_text().strip().splitlines()
    assert len(rows) == 3 and rows[1].startswith("conv,1,2,") and rows[2].split(",")[8] == "true"
    assert run_suite(BenchConfig("brgemm", iters=2, baseline=True)) == 0
    assert run_suite(BenchConfig("fc", minibatch=128, c=256, k=256, iters=2)) == 0
    assert run_suite(BenchConfig("lstm", minibatch=8, c=128, k=128, t_steps=3, iters=1)) == 0
    text = capsys.readouterr().out
    assert "brgemm_baseline,0,1," in text and "fc,0,128," in text and "lstm,0,8," in text
