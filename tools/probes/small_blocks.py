"""Probe: where the small-block (m = 32) generic BRGEMM and the LstmDP step spend time."""
import json
import os
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch  # noqa: E402

from paper_1906_06440_b200 import _lib  # noqa: E402

lib = _lib.load()


def tm(fn, iters=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


out = {}
for (m, batch, jobs, notma) in [(32, 16, 1184, 0), (32, 16, 4736, 0), (32, 1, 1184, 0), (32, 64, 1184, 0),
                                (64, 16, 1184, 0), (64, 16, 1184, 1), (64, 1, 1184, 1), (128, 16, 1184, 1)]:
    n = k = m
    if notma:
        os.environ["BRK_GENERIC_NO_TMA"] = "1"
    else:
        os.environ.pop("BRK_GENERIC_NO_TMA", None)
    a = torch.randn(jobs * batch * k * m, device="cuda").bfloat16()
    b = torch.randn(jobs * batch * n * k, device="cuda").bfloat16()
    c = torch.empty(jobs * n * m, device="cuda")
    fn = lambda: _lib.check(lib.brk_brgemm_stride(a.data_ptr(), b.data_ptr(), k * m, n * k, c.data_ptr(), jobs,  # noqa
                                                  batch * k * m, batch * n * k, n * m, m, n, k, batch, m, k, m, 1.0,
                                                  0.0, _lib.BRK_BF16, _lib.BRK_F32, _lib.BRK_COMPUTE_BF16, 0))
    us = tm(fn)
    byts = jobs * (2 * batch * (m * k + k * n) + 4 * m * n)
    out[f"m{m}_b{batch}_j{jobs}_notma{notma}"] = {"us": us, "GBs": byts / us / 1e3,
                                                 "us_per_stage_per_cta": us / (jobs * batch / 148)}
    print(json.dumps({f"m{m}_b{batch}_j{jobs}_notma{notma}": out[f"m{m}_b{batch}_j{jobs}_notma{notma}"]}), flush=True)
os.environ.pop("BRK_GENERIC_NO_TMA", None)

# LstmDP breakdown
from paper_1906_06440_b200 import precision  # noqa: E402
from paper_1906_06440_b200.lstm import lstm_backward, lstm_forward  # noqa: E402
from paper_1906_06440_b200.train import LstmDP  # noqa: E402

net = LstmDP()
p = net.params
with precision("bf16"):
    def fb():
        seq = lstm_forward(p, net.x)
        lstm_backward(p, net.x, seq, net.dh)
    out["lstm_api_fwd_bwd_cached_us"] = tm(fb, 5)
    out["lstm_dp_step_us"] = tm(net.step, 5)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        net.step()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    out["lstm_dp_step_host_us"] = (t1 - t0) / 5 * 1e6
    from paper_1906_06440_b200.lstm import _device_cell, _seq_cell  # noqa: E402

    def rebuild():
        object.__setattr__(p, "_brk_device_cell", None)
        _seq_cell(p)
    out["lstm_cell_rebuild_us"] = tm(rebuild, 5)
print(json.dumps(out), flush=True)
