"""Cross-check the oracle's restated backward passes (no reference path exists)
against torch.autograd in float64 on CPU."""

import numpy as np
import torch

import brk_oracle as orc


def _t(a):
    return torch.tensor(np.asarray(a, np.float64), dtype=torch.float64, requires_grad=True)


def test_fc_backward_vs_autograd():
    rng = np.random.default_rng(0)
    n, c, k = 12, 10, 8
    w = rng.uniform(-1, 1, (k, c)).astype(np.float32)
    x = rng.uniform(-1, 1, (n, c)).astype(np.float32)
    b = rng.uniform(-1, 1, k).astype(np.float32)
    dy = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    for act in ("identity", "relu", "sigmoid"):
        y = orc.fc_forward_reference(w, x.T, act, b).T
        dx, dw, db = orc.fc_backward_reference(w, x, y, dy, act)
        tw, tx, tb = _t(w), _t(x), _t(b)
        z = tx @ tw.T + tb
        out = {"identity": z, "relu": torch.relu(z), "sigmoid": torch.sigmoid(z)}[act]
        out.backward(torch.tensor(dy, dtype=torch.float64))
        assert np.allclose(dx, tx.grad.numpy(), atol=1e-5)
        assert np.allclose(dw, tw.grad.numpy(), atol=1e-5)
        assert np.allclose(db, tb.grad.numpy(), atol=1e-5)


def test_fc_blocked_backward_equals_dense():
    from paper_1906_06440_b200.tensor import block_fc_activation, block_weight_2d

    rng = np.random.default_rng(1)
    n, c, k = 16, 24, 32
    w = rng.uniform(-1, 1, (k, c)).astype(np.float32)
    x = rng.uniform(-1, 1, (n, c)).astype(np.float32)
    y = orc.fc_forward_reference(w, x.T, "relu").T.copy()
    dy = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    dx, dw, db = orc.fc_backward_reference(w, x, y, dy, "relu")
    dxb, dwb, dbb = orc.fc_backward_blocked(block_weight_2d(w, 8, 16).data, block_fc_activation(x, 4, 8).data,
                                            block_fc_activation(y, 4, 16).data, block_fc_activation(dy, 4, 16).data,
                                            "relu")
    assert np.allclose(dxb.transpose(0, 2, 1, 3).reshape(n, c), dx, atol=1e-6)
    assert np.allclose(dwb.transpose(0, 3, 1, 2).reshape(k, c), dw, atol=1e-6)
    assert np.allclose(dbb, db, atol=1e-6)


def test_mlp_step_vs_autograd():
    rng = np.random.default_rng(2)
    n, c, layers = 16, 8, 3
    ws = [rng.uniform(-1, 1, (c, c)).astype(np.float32) / 3 for _ in range(layers)]
    bs = [rng.uniform(-0.1, 0.1, c).astype(np.float32) for _ in range(layers)]
    x = rng.uniform(-1, 1, (n, c)).astype(np.float32)
    dy = rng.uniform(-1, 1, (n, c)).astype(np.float32)
    out = orc.mlp_step_reference(ws, bs, x, dy, lr=0.1)
    tws = [_t(w) for w in ws]
    tbs = [_t(b) for b in bs]
    tx = _t(x)
    h = tx
    for tw, tb in zip(tws, tbs):
        h = torch.relu(h @ tw.T + tb)
    h.backward(torch.tensor(dy, dtype=torch.float64))
    for l in range(layers):
        assert np.allclose(out["dw"][l], tws[l].grad.numpy(), atol=1e-5)
        assert np.allclose(out["db"][l], tbs[l].grad.numpy(), atol=1e-5)
        assert np.allclose(out["w_new"][l], ws[l] - 0.1 * tws[l].grad.numpy(), atol=1e-5)
    assert np.allclose(out["dx"], tx.grad.numpy(), atol=1e-5)


def test_lstm_backward_vs_autograd():
    rng = np.random.default_rng(3)
    t_steps, n, c, k = 4, 3, 5, 6
    sc = 1 / np.sqrt(c + k)
    w = {g: (rng.uniform(-1, 1, (k, c)) * sc).astype(np.float32) for g in orc.GATES}
    r = {g: (rng.uniform(-1, 1, (k, k)) * sc).astype(np.float32) for g in orc.GATES}
    b = {g: (rng.uniform(-1, 1, k) * sc).astype(np.float32) for g in orc.GATES}
    x = rng.uniform(-1, 1, (t_steps, n, c)).astype(np.float32)
    h0 = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    s0 = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    dh = rng.uniform(-1, 1, (t_steps, n, k)).astype(np.float32)
    fwd = orc.lstm_forward_reference(w, r, b, x, h0, s0)
    bwd = orc.lstm_backward_reference(w, r, x, fwd, dh, h0, s0)
    tw = {g: _t(w[g]) for g in orc.GATES}
    tr = {g: _t(r[g]) for g in orc.GATES}
    tb = {g: _t(b[g]) for g in orc.GATES}
    tx = _t(x)
    th0, ts0 = _t(h0), _t(s0)
    h, s = th0, ts0
    hs = []
    for t in range(t_steps):
        pre = {g: tx[t] @ tw[g].T + h @ tr[g].T + tb[g] for g in orc.GATES}
        i, cc, f, o = torch.sigmoid(pre["i"]), torch.tanh(pre["c"]), torch.sigmoid(pre["f"]), torch.sigmoid(pre["o"])
        s = f * s + i * cc
        h = o * torch.tanh(s)
        hs.append(h)
    torch.stack(hs).backward(torch.tensor(dh, dtype=torch.float64))
    # the oracle uses f32-rounded stored states, autograd carries f64: compare at 1e-5
    assert np.allclose(bwd["dx"], tx.grad.numpy(), atol=1e-5)
    for g in orc.GATES:
        assert np.allclose(bwd["dw"][g], tw[g].grad.numpy(), atol=1e-5)
        assert np.allclose(bwd["dr"][g], tr[g].grad.numpy(), atol=1e-5)
        assert np.allclose(bwd["db"][g], tb[g].grad.numpy(), atol=1e-5)
    assert np.allclose(bwd["dh0"], th0.grad.numpy(), atol=1e-5)
    assert np.allclose(bwd["ds0"], ts0.grad.numpy(), atol=1e-5)


def test_conv_backward_vs_autograd():
    rng = np.random.default_rng(4)
    for (n, c, k, h, w_, r, stride) in [(2, 3, 4, 7, 6, 3, 1), (1, 4, 5, 9, 8, 3, 2), (2, 3, 2, 8, 8, 1, 2),
                                        (1, 2, 3, 11, 9, 7, 2)]:
        i = rng.uniform(-1, 1, (n, c, h, w_)).astype(np.float32)
        wt = rng.uniform(-1, 1, (k, c, r, r)).astype(np.float32)
        pad = (r - 1) // 2
        o = orc.conv2d_forward_reference(i, wt, stride)
        do = rng.uniform(-1, 1, o.shape).astype(np.float32)
        di = orc.conv2d_backward_data_reference(do, wt, (h, w_), stride)
        dw = orc.conv2d_weight_update_reference(i, do, r, r, stride)
        ti, tw = _t(i), _t(wt)
        to = torch.nn.functional.conv2d(ti, tw, stride=stride, padding=pad)
        assert np.allclose(o, to.detach().numpy(), atol=1e-5)
        to.backward(torch.tensor(do, dtype=torch.float64))
        assert np.allclose(di, ti.grad.numpy(), atol=1e-5)
        assert np.allclose(dw, tw.grad.numpy(), atol=1e-4)
