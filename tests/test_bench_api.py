"""The reference measurement API (brkernels.bench: FLOP accounting, ResNet-50 table,
weighted efficiency, layer parsing, CLI) — host logic, no GPU."""

import pytest

from paper_1906_06440_b200.bench import (
    CSV_HEADER,
    BenchResult,
    _build_parser,
    flops_brgemm,
    flops_conv,
    flops_fc,
    flops_lstm_fwd,
    parse_layers,
    resnet50_table,
    weighted_efficiency,
)
from paper_1906_06440_b200.brgemm import BrgemmSpec


def test_resnet50_table_has_53_convs_and_reference_flops():
    table = resnet50_table(28)
    assert len(table) == 20 and sum(r.count for r in table) == 53
    stem = table[0].spec
    assert (stem.c, stem.k, stem.r, stem.stride, stem.out_h) == (3, 64, 7, 2, 112)
    assert flops_conv(stem, 28) == 2 * 28 * 64 * 3 * 49 * 112 * 112
    assert flops_lstm_fwd(50, 168, 1024, 1024) == 2 * 50 * 168 * 8 * 1024 * 1024
    assert flops_fc(2048, 1024, 1024) == 2 * 2048 * 1024 * 1024
    assert flops_brgemm(BrgemmSpec(m=64, n=64, k=64, batch=16)) == 2 * 64 ** 3 * 16


def test_weighted_efficiency_and_parse_layers():
    res = [(BenchResult(100, 1.0, 0.5, 1, 1), 2), (BenchResult(50, 0.5, 0.5, 1, 1), 1)]
    assert weighted_efficiency(res, 100.0) == pytest.approx(250 / 2.5 / 100)
    with pytest.raises(ValueError):
        weighted_efficiency([], 1.0)
    with pytest.raises(ValueError):
        BenchResult(1, 0.0, 1.0, 1, 1)
    assert parse_layers("1,4,8-10") == [1, 4, 8, 9, 10]
    with pytest.raises(ValueError):
        parse_layers("0-3")


def test_cli_mirrors_reference_flags():
    p = _build_parser()
    a = p.parse_args(["conv", "--layers", "2-5", "--minibatch", "4", "--iters", "3", "--csv", "x.csv"])
    assert (a.workload, a.layers, a.minibatch, a.iters, a.csv) == ("conv", "2-5", 4, 3, "x.csv")
    a = p.parse_args(["brgemm", "--m", "32", "--k", "16", "--baseline"])
    assert (a.m, a.k_dim, a.baseline, a.minibatch_default) == (32, 16, True, 1)
    assert CSV_HEADER.startswith("workload,id,N,workers,flops,seconds_mean,seconds_min,gflops,verified")
