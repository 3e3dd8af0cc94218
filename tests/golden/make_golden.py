"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``brkernels`` read-only from
/root/reference/pkg/src, evaluates it on small seeded inputs mirroring the
reference's own tests (seeds/generators cited per case) and writes compact
.npz fixtures next to this file.  The fixtures travel with the repo; nothing
at test time reads /root/reference.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
F32 = np.float32


def _ref():
    sys.path.insert(0, str(REF_SRC))
    import brkernels  # noqa: F401  (the reference package, unmodified)

    return brkernels


def brgemm_cases(bk):
    """Acceptance-style generator (tests/test_acceptance.py:50-86), shrunk extents."""
    rng = np.random.default_rng(2024_08)
    out = {}
    for trial in range(48):
        m = int(rng.integers(1, 80))
        n = int(rng.integers(1, 80))
        k = int(rng.integers(1, 96))
        batch = int(rng.integers(0, 5))
        beta = float(rng.integers(0, 2))
        integer = trial % 3 == 0
        draw = (lambda s: rng.integers(-2, 3, size=s).astype(F32)) if integer else \
            (lambda s: rng.uniform(-1, 1, size=s).astype(F32))
        a = np.stack([draw((k, m)) for _ in range(batch)]) if batch else np.zeros((0, k, m), F32)
        b = np.stack([draw((n, k)) for _ in range(batch)]) if batch else np.zeros((0, n, k), F32)
        c0 = draw((n, m))
        spec = bk.BrgemmSpec(m=m, n=n, k=k, batch=batch, alpha=1.0, beta=beta)
        got = bk.brgemm(list(a), list(b), c0.copy(), spec, bk.plan_tiles(m, n))
        ref = bk.brgemm_reference(list(a), list(b), c0.copy(), spec)
        out[f"t{trial}"] = dict(a=a, b=b, c0=c0, beta=np.float64(beta), integer=np.int8(integer),
                                tiled=got, oracle=ref)
    # strided variant (tests/test_brgemm.py:132-160)
    rng = np.random.default_rng(7)
    a_stack = rng.uniform(-1, 1, (4, 6, 8)).astype(F32)
    b_stack = rng.uniform(-1, 1, (4, 5, 6)).astype(F32)
    spec = bk.BrgemmSpec(m=8, n=5, k=6, batch=4, beta=0.0)
    out["strided"] = dict(a=a_stack, b=b_stack,
                          got=bk.brgemm_strided(a_stack, b_stack, 48, 30, np.zeros((5, 8), F32), spec))
    # alpha/beta edge cases (tests/test_brgemm.py:45-58, 105-112)
    rng = np.random.default_rng(6)
    a0 = rng.uniform(-1, 1, (3, 4)).astype(F32)
    b0 = rng.uniform(-1, 1, (2, 3)).astype(F32)
    c0 = rng.uniform(-1, 1, (2, 4)).astype(F32)
    spec = bk.BrgemmSpec(m=4, n=2, k=3, batch=3, alpha=2.0, beta=1.0)
    out["zero_stride"] = dict(a=a0, b=b0, c0=c0, got=bk.brgemm_strided(a0, b0, 0, 0, c0.copy(), spec))
    return out


def planner_cases(bk):
    rows = []
    for vlen in (4, 8, 16):
        for budget in (16, 32):
            for m in range(1, 129, 7):
                for n in range(1, 33, 5):
                    p = bk.plan_tiles(m, n, vlen=vlen, budget=budget)
                    rows.append((m, n, vlen, budget, p.m_b, p.n_b, p.accumulators, int(p.degraded)))
    return np.asarray(rows, np.int64)


def fc_cases(bk):
    out = {}
    for ck in (128, 256):  # tests/test_acceptance.py:155-168 (N=64), C=K shrunk
        rng = np.random.default_rng([33, ck])
        w = rng.uniform(-1, 1, (ck, ck)).astype(F32)
        x = rng.uniform(-1, 1, (64, ck)).astype(F32)
        for act in bk.Activation:
            params = bk.FcParams.from_dense(w, 64, activation=act)
            xb = bk.block_fc_activation(x, params.b_n, params.b_c)
            y = bk.unblock_fc_activation(bk.fc_forward(params, xb))
            ref = np.ascontiguousarray(bk.fc_forward_reference(w, x.T, act).T)
            out[f"ck{ck}_{act.value}"] = dict(w=w, x=x, y=y, oracle=ref)
    # identity-weights KAT (tests/test_fc.py:50-56)
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (8, 16)).astype(F32)
    params = bk.FcParams.from_dense(np.eye(16, dtype=F32), 8, b_n=4, b_c=8, b_k=8)
    y = bk.unblock_fc_activation(bk.fc_forward(params, bk.block_fc_activation(x, 4, 8)))
    out["identity"] = dict(x=x, y=y)
    # integer-valued FC KAT (exact in bf16/tf32)
    rng = np.random.default_rng(35)
    w = rng.integers(-2, 3, (128, 128)).astype(F32)
    x = rng.integers(-2, 3, (128, 128)).astype(F32)
    params = bk.FcParams.from_dense(w, 128, activation=bk.Activation.RELU)
    y = bk.unblock_fc_activation(bk.fc_forward(params, bk.block_fc_activation(x, params.b_n, params.b_c)))
    out["int_relu"] = dict(w=w, x=x, y=y)
    return out


def lstm_cases(bk):
    out = {}
    for ck in (64, 128):  # tests/test_acceptance.py:132-152
        rng = np.random.default_rng([22, ck])
        weights = bk.LstmCellWeights.random(rng, ck, ck)
        x = rng.uniform(-1, 1, (8, 8, ck)).astype(F32)
        params = bk.LstmParams.from_dense(weights, 8, 8)
        seq = bk.lstm_forward(params, x, keep_gates=True)
        ref = bk.lstm_forward_reference(weights, x, keep_gates=True)
        d = dict(x=x, h=seq.h, s=seq.s, h_oracle=ref.h, s_oracle=ref.s)
        for g in ("i", "c", "f", "o"):
            d[f"w_{g}"] = getattr(weights, f"w_{g}")
            d[f"r_{g}"] = getattr(weights, f"r_{g}")
            d[f"bias_{g}"] = getattr(weights, f"bias_{g}")
            d[f"gate_{g}"] = seq.gates[g]
        out[f"ck{ck}"] = d
    # nonzero initial state (tests/test_lstm.py:150-158)
    rng = np.random.default_rng(4)
    weights = bk.LstmCellWeights.random(np.random.default_rng(4), 8, 8)
    x = np.random.default_rng(4).uniform(-1, 1, (2, 4, 8)).astype(F32)
    h0 = rng.uniform(-1, 1, (4, 8)).astype(F32)
    s0 = rng.uniform(-1, 1, (4, 8)).astype(F32)
    ref = bk.lstm_forward_reference(weights, x, h_init=h0, s_init=s0)
    d = dict(x=x, h0=h0, s0=s0, h_oracle=ref.h, s_oracle=ref.s)
    for g in ("i", "c", "f", "o"):
        d[f"w_{g}"] = getattr(weights, f"w_{g}")
        d[f"r_{g}"] = getattr(weights, f"r_{g}")
        d[f"bias_{g}"] = getattr(weights, f"bias_{g}")
    out["init_state"] = d
    return out


def conv_cases(bk):
    out = {}
    rng = np.random.default_rng(2024_11)  # tests/test_acceptance.py:106-128
    for trial in range(24):
        rs = int(rng.choice([1, 3, 7]))
        stride = int(rng.choice([1, 2]))
        h = int(rng.integers(max(2, rs - 2), 13))
        w = int(rng.integers(max(2, rs - 2), 13))
        c = int(rng.integers(1, 33))
        k = int(rng.integers(1, 33))
        n = int(rng.integers(1, 3))
        spec = bk.ConvSpec(n=n, c=c, k=k, h=h, w=w, r=rs, s=rs, stride=stride)
        i_dense = rng.uniform(-1, 1, (n, c, h, w)).astype(F32)
        w_dense = rng.uniform(-1, 1, (k, c, rs, rs)).astype(F32)
        inp, wgt = bk.block_conv_tensors(i_dense, w_dense, spec.b_c, spec.b_k)
        got = bk.unblock_conv_output(bk.conv2d_forward(spec, inp, wgt))
        ref = bk.conv2d_forward_reference(spec, i_dense, w_dense)
        out[f"t{trial}"] = dict(i=i_dense, w=w_dense, stride=np.int64(stride), got=got, oracle=ref)
    # integer 7-loop KATs (tests/test_cnn.py:97-114)
    rng = np.random.default_rng(2)
    spec = bk.ConvSpec(n=2, c=3, k=4, h=7, w=7, r=3, s=3, stride=2, b_c=3, b_k=4)
    i_dense = rng.integers(-2, 3, (2, 3, 7, 7)).astype(F32)
    w_dense = rng.integers(-2, 3, (4, 3, 3, 3)).astype(F32)
    out["int_stride2"] = dict(i=i_dense, w=w_dense, stride=np.int64(2),
                              oracle=bk.conv2d_forward_reference(spec, i_dense, w_dense))
    # ResNet-50-shaped layers with channels/spatial shrunk 4x (table bench.py:57-79)
    for lid, c, k, h, w, r, s, stride, _ in bk.bench._RESNET50_ROWS:
        if lid not in (1, 2, 4, 6, 13, 18):
            continue
        c2, k2 = max(3, c // 8) if lid == 1 else c // 8, k // 8
        h2, w2 = max(7, h // 8), max(7, w // 8)
        spec = bk.ConvSpec(n=2, c=c2, k=k2, h=h2, w=w2, r=r, s=s, stride=stride)
        rng = np.random.default_rng([11, lid])
        i_dense = rng.uniform(-1, 1, (2, c2, h2, w2)).astype(F32)
        w_dense = rng.uniform(-1, 1, (k2, c2, r, s)).astype(F32)
        out[f"resnet{lid}"] = dict(i=i_dense, w=w_dense, stride=np.int64(stride),
                                   oracle=bk.conv2d_forward_reference(spec, i_dense, w_dense))
    return out


def tensor_cases(bk):
    rng = np.random.default_rng(9)
    w = rng.uniform(-1, 1, (8, 12)).astype(F32)
    x = rng.uniform(-1, 1, (6, 12)).astype(F32)
    i = rng.uniform(-1, 1, (2, 6, 3, 4)).astype(F32)
    kw = rng.uniform(-1, 1, (4, 6, 3, 3)).astype(F32)
    bi, bw = bk.block_conv_tensors(i, kw, 3, 2)
    padded = bk.pad_spatial(bi, 1, 2)
    return dict(w=w, x=x, i=i, kw=kw,
                w_blk=bk.block_weight_2d(w, 4, 2).data,
                x_blk=bk.block_fc_activation(x, 3, 4).data,
                i_blk=bi.data, kw_blk=bw.data, i_pad=padded.data,
                mre=np.float64(bk.max_rel_error(x, x + 1e-3)))


def save(name, cases):
    flat = {}
    if isinstance(cases, dict):
        for key, val in cases.items():
            if isinstance(val, dict):
                for k2, v2 in val.items():
                    flat[f"{key}__{k2}"] = np.asarray(v2)
            else:
                flat[key] = np.asarray(val)
    else:
        flat["rows"] = cases
    np.savez_compressed(OUT / f"{name}.npz", **flat)
    print(f"wrote {name}.npz ({(OUT / f'{name}.npz').stat().st_size / 1024:.0f} KiB)")


def main():
    bk = _ref()
    import brkernels.bench  # noqa: F401  (table rows)

    save("brgemm", brgemm_cases(bk))
    save("planner", planner_cases(bk))
    save("fc", fc_cases(bk))
    save("lstm", lstm_cases(bk))
    save("conv", conv_cases(bk))
    save("tensor", tensor_cases(bk))


if __name__ == "__main__":
    main()
