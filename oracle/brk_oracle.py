"""CPU oracle for the BRGEMM hot path — TEST INFRASTRUCTURE, NOT THE PRODUCT.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module, and only as the checker or
the timed CPU arm.  The product package ``paper_1906_06440_b200`` never
imports it and has no CPU fallback.

Restated from the reference package ``brkernels`` (pure Python/NumPy, read at
/root/reference/pkg/src/brkernels; every function cites the file:line it
follows).  Precision follows the reference: float32 storage, float64
accumulation, one float32 rounding of each stored result.

Parity pinning: the forward functions here are checked bit-for-bit (integer
KATs) and to 1e-12 (random inputs) against golden vectors produced by running
the reference itself (tests/golden/make_golden.py -> tests/golden/*.npz, test
tests/test_oracle_golden.py).  The backward-data / weight-update / bias / BPTT
passes have no reference implementation (the reference is forward-only,
README.md:117-121); they are restated from the forward definitions and
cross-checked against torch.autograd in float64 (tests/test_oracle_autograd.py).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

F32 = np.float32
F64 = np.float64
GATES = ("i", "c", "f", "o")  # reference lstm.py:28


# ---------------------------------------------------------------------------
# rounding emulation (for predicted-error checks of the TF32/BF16 tensor-core path)
# ---------------------------------------------------------------------------
def round_bf16(x) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 -> float32."""
    u = np.ascontiguousarray(x, dtype=F32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(F32)


def round_tf32(x) -> np.ndarray:
    """Round-to-nearest (ties away, cvt.rna) float32 -> tf32 (10-bit mantissa) -> float32."""
    u = np.ascontiguousarray(x, dtype=F32).view(np.uint32).astype(np.uint64)
    u = (u + 0x1000) & 0xFFFFE000
    return u.astype(np.uint32).view(F32)


def scale_rel_error(got, ref) -> float:
    """max|got-ref| / max|ref| — the TF32 (1e-3) / BF16 (1e-2) tolerance metric."""
    g = np.asarray(got, F64)
    r = np.asarray(ref, F64)
    if r.size == 0:
        return 0.0
    return float(np.max(np.abs(g - r)) / max(float(np.max(np.abs(r))), 1e-30))


def max_rel_error(a, b) -> float:
    """Elementwise |a-b| / max(|b|, 1e-6) (reference tensor.py:278-286)."""
    a = np.asarray(a, F64)
    b = np.asarray(b, F64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-6)))


# ---------------------------------------------------------------------------
# BRGEMM (reference brgemm.py)
# ---------------------------------------------------------------------------
def brgemm_reference(a_blocks, b_blocks, c, alpha=1.0, beta=1.0):
    """C = alpha * sum_i B_i @ A_i + beta * C, float64 sum, one f32 round (brgemm.py:210-225).

    a_blocks[i]: (k, m); b_blocks[i]: (n, k); c: (n, m).  Returns a new array.
    """
    c = np.asarray(c, F32)
    total = np.zeros(c.shape, F64)
    if alpha != 0.0:
        for a, b in zip(a_blocks, b_blocks):
            total += np.asarray(b, F64) @ np.asarray(a, F64)
        total *= alpha
    if beta != 0.0:
        total += beta * c.astype(F64)
    return total.astype(F32)


def strided_blocks(base, stride: int, rows: int, cols: int, batch: int):
    """Blocks at i*stride of the flattened base (brgemm.py:296-337)."""
    flat = np.ravel(base)
    span = rows * cols
    return [flat[i * stride: i * stride + span].reshape(rows, cols) for i in range(batch)]


def offset_blocks(base, offsets, rows: int, cols: int):
    """Offset variant (north star): block i starts at element offsets[i]."""
    flat = np.ravel(base)
    span = rows * cols
    return [flat[o: o + span].reshape(rows, cols) for o in offsets]


def plan_tiles_reference(m, n, vlen=16, fma_latency=5, budget=32):
    """Exhaustive register-tile search (the planner's specification, tests/test_brgemm.py:201-219)."""
    mbs = [m] if m < vlen else [v * vlen for v in range(1, m // vlen + 1)]
    best = None
    for m_b in mbs:
        for n_b in range(1, n + 1):
            acc = n_b * -(-m_b // vlen)
            if acc + n_b + 1 > budget:
                continue
            key = (acc, m % m_b == 0, m_b, n_b)
            if best is None or key > best:
                best = key
    if best is None:
        return None
    acc, _, m_b, n_b = best
    return m_b, n_b, acc, acc < fma_latency


# ---------------------------------------------------------------------------
# FC (reference fc.py)
# ---------------------------------------------------------------------------
def _act(z, activation: str):
    if activation == "relu":
        return np.maximum(z, 0.0)
    if activation == "sigmoid":
        return 1.0 / (1.0 + np.exp(-z))
    return z


def _act_grad(y, activation: str):
    """g'(z) expressed through y = g(z)."""
    if activation == "relu":
        return (y > 0).astype(F64)
    if activation == "sigmoid":
        return y * (1.0 - y)
    return np.ones_like(y)


def fc_forward_reference(w, x, activation="identity", bias=None):
    """Y = g(W @ X (+ b)) with W (K, C), X (C, N); float64, one f32 round (fc.py:166-179).

    ``bias`` (K,) is the north-star extension (the reference has none, fc.py:5).
    """
    z = np.asarray(w, F64) @ np.asarray(x, F64)
    if bias is not None:
        z = z + np.asarray(bias, F64)[:, None]
    return _act(z, activation).astype(F32)


def fc_backward_reference(w, x, y, dy, activation="identity"):
    """Backward of Y = g(W X + b) (no reference path; restated).

    Shapes: w (K, C), x (N, C), y/dy (N, K).  Returns dx (N, C), dw (K, C), db (K,)
    computed from dz = dy * g'(z) in float64, rounded once to f32.
    """
    dz = np.asarray(dy, F64) * _act_grad(np.asarray(y, F64), activation)
    dx = dz @ np.asarray(w, F64)
    dw = dz.T @ np.asarray(x, F64)
    db = dz.sum(axis=0)
    return dx.astype(F32), dw.astype(F32), db.astype(F32)


def fc_forward_blocked(w_blk, x_blk, activation="identity", bias=None, workers=1):
    """The reference's blocked FC algorithm (fc.py:99-163 over brgemm.py:260-293).

    w_blk [K_b][C_b][b_c][b_k], x_blk [N_b][C_b][b_n][b_c] -> y [N_b][K_b][b_n][b_k].
    Per output block: float64 accumulation of the C_b block products, one f32
    store, activation on the hot block; items ib_k-major / ib_n-minor split over
    ``workers`` threads (partition.py:24-50).  Used as the timed CPU arm.
    """
    k_b, c_b, b_c, b_k = w_blk.shape
    n_b, _, b_n, _ = x_blk.shape
    y = np.empty((n_b, k_b, b_n, b_k), F32)
    w64 = w_blk.astype(F64)
    x64 = x_blk.astype(F64)

    def item(flat):
        ib_k, ib_n = divmod(flat, n_b)
        acc = np.zeros((b_n, b_k), F64)
        for cb in range(c_b):
            acc += x64[ib_n, cb] @ w64[ib_k, cb]
        if bias is not None:
            acc += np.asarray(bias, F64)[ib_k * b_k:(ib_k + 1) * b_k]
        y[ib_n, ib_k] = _act(acc, activation)

    _run_items(item, k_b * n_b, workers)
    return y


def _run_items(fn, count, workers):
    if workers <= 1:
        for i in range(count):
            fn(i)
        return
    chunk = math.ceil(count / workers)
    with ThreadPoolExecutor(max_workers=workers) as pool:
        list(pool.map(lambda w0: [fn(i) for i in range(w0, min(count, w0 + chunk))],
                      range(0, count, chunk)))


def fc_backward_blocked(w_blk, x_blk, y_blk, dy_blk, activation="identity", workers=1):
    """Blocked bwd-data / weight-update / bias passes in the same loop style (restated)."""
    k_b, c_b, b_c, b_k = w_blk.shape
    n_b, _, b_n, _ = x_blk.shape
    dz = dy_blk.astype(F64) * _act_grad(y_blk.astype(F64), activation)
    w64 = w_blk.astype(F64)
    x64 = x_blk.astype(F64)
    dx = np.empty((n_b, c_b, b_n, b_c), F32)
    dw = np.empty((k_b, c_b, b_c, b_k), F32)

    def item_dx(flat):
        ib_c, ib_n = divmod(flat, n_b)
        acc = np.zeros((b_n, b_c), F64)
        for kb in range(k_b):
            acc += dz[ib_n, kb] @ w64[kb, ib_c].T
        dx[ib_n, ib_c] = acc

    def item_dw(flat):
        ib_k, ib_c = divmod(flat, c_b)
        acc = np.zeros((b_c, b_k), F64)
        for nb in range(n_b):
            acc += x64[nb, ib_c].T @ dz[nb, ib_k]
        dw[ib_k, ib_c] = acc

    _run_items(item_dx, c_b * n_b, workers)
    _run_items(item_dw, k_b * c_b, workers)
    db = dz.sum(axis=(0, 2)).reshape(-1).astype(F32)
    return dx, dw, db


def mlp_step_reference(ws, bs, x, dy, lr=0.0, store=None, activations=None):
    """One MLP step (forward, backward-data, weight update, SGD) in float64.

    ws[l] (K, C), bs[l] (K,), x (N, C), dy (N, K_last) — ReLU after every layer.
    Stored tensors (activations y_l and back-propagated dz_l) are rounded to
    float32, then by ``store`` (e.g. ``round_bf16`` to mirror a bf16-storage
    implementation) at the same points an implementation stores them.
    ``activations`` (optional list y_1..y_L) replaces the forward pass so the
    backward pass uses exactly the implementation's ReLU masks (activations
    within rounding of 0 otherwise flip masks between implementations).
    Returns dict(y=[...], dx, dw=[...], db=[...], w_new, b_new).
    """
    rnd = (lambda a: np.asarray(a, F32)) if store is None else (lambda a: store(np.asarray(a, F32)))
    ys = [rnd(x)]
    if activations is not None:
        ys.extend(np.asarray(a, F32) for a in activations)
    else:
        for w, b in zip(ws, bs):
            ys.append(rnd(fc_forward_reference(w, ys[-1].T, "relu", b).T.copy()))
    dz = np.asarray(dy, F64) * (ys[-1] > 0)
    dws, dbs = [None] * len(ws), [None] * len(ws)
    dx = None
    for l in range(len(ws) - 1, -1, -1):
        dws[l] = (dz.T @ ys[l].astype(F64)).astype(F32)
        dbs[l] = dz.sum(axis=0).astype(F32)
        g = dz @ np.asarray(ws[l], F64)
        if l > 0:
            dz = rnd(g * (ys[l] > 0)).astype(F64)
        else:
            dx = rnd(g)
    w_new = [(np.asarray(w, F64) - lr * dw).astype(F32) for w, dw in zip(ws, dws)]
    b_new = [(np.asarray(b, F64) - lr * db).astype(F32) for b, db in zip(bs, dbs)]
    return {"y": ys, "dx": dx, "dw": dws, "db": dbs, "w_new": w_new, "b_new": b_new}


# ---------------------------------------------------------------------------
# LSTM (reference lstm.py)
# ---------------------------------------------------------------------------
def _sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def lstm_forward_reference(w, r, b, x, h0=None, s0=None):
    """Whole-matrix LSTM forward, float64 within a step, f32 h/s between steps (lstm.py:330-378).

    w[g] (K, C), r[g] (K, K), b[g] (K,) for g in (i, c, f, o); x (T, N, C).
    Returns dict(h, s, gates={g: (T, N, K)}) — all float32.
    """
    t_steps, n, _ = x.shape
    k = w["i"].shape[0]
    h_prev = np.zeros((n, k)) if h0 is None else np.asarray(h0, F64)
    s_prev = np.zeros((n, k)) if s0 is None else np.asarray(s0, F64)
    h = np.empty((t_steps, n, k), F32)
    s = np.empty((t_steps, n, k), F32)
    gates = {g: np.empty((t_steps, n, k), F32) for g in GATES}
    w64 = {g: np.asarray(w[g], F64) for g in GATES}
    r64 = {g: np.asarray(r[g], F64) for g in GATES}
    b64 = {g: np.asarray(b[g], F64) for g in GATES}
    for t in range(t_steps):
        xt = np.asarray(x[t], F64)
        pre = {g: xt @ w64[g].T + h_prev @ r64[g].T + b64[g] for g in GATES}
        gi, gc, gf, go = _sigmoid(pre["i"]), np.tanh(pre["c"]), _sigmoid(pre["f"]), _sigmoid(pre["o"])
        st = gf * s_prev + gi * gc
        ht = go * np.tanh(st)
        h[t], s[t] = ht, st
        for g, v in zip(GATES, (gi, gc, gf, go)):
            gates[g][t] = v
        h_prev = h[t].astype(F64)
        s_prev = s[t].astype(F64)
    return {"h": h, "s": s, "gates": gates}


def lstm_backward_reference(w, r, x, fwd, dh, h0=None, s0=None):
    """BPTT for the reference cell equations (no reference path; restated).

    Uses the forward's stored f32 gates/h/s (as a fused kernel would).
    dh: (T, N, K) gradient w.r.t. every h_t.  Returns float32
    dict(dx (T,N,C), dw{g}, dr{g}, db{g}, dh0, ds0).
    """
    t_steps, n, c = x.shape
    k = w["i"].shape[0]
    w64 = {g: np.asarray(w[g], F64) for g in GATES}
    r64 = {g: np.asarray(r[g], F64) for g in GATES}
    gate = {g: fwd["gates"][g].astype(F64) for g in GATES}
    h = fwd["h"].astype(F64)
    s = fwd["s"].astype(F64)
    h_init = np.zeros((n, k)) if h0 is None else np.asarray(h0, F64)
    s_init = np.zeros((n, k)) if s0 is None else np.asarray(s0, F64)
    dw = {g: np.zeros((k, c)) for g in GATES}
    dr = {g: np.zeros((k, k)) for g in GATES}
    db = {g: np.zeros(k) for g in GATES}
    dx = np.zeros((t_steps, n, c))
    dh_next = np.zeros((n, k))
    ds_next = np.zeros((n, k))
    for t in range(t_steps - 1, -1, -1):
        gi, gc, gf, go = (gate[g][t] for g in GATES)
        s_prev = s[t - 1] if t > 0 else s_init
        h_prev = h[t - 1] if t > 0 else h_init
        tanh_s = np.tanh(s[t])
        dht = np.asarray(dh[t], F64) + dh_next
        ds = dht * go * (1.0 - tanh_s ** 2) + ds_next
        dpre = {
            "i": ds * gc * gi * (1.0 - gi),
            "c": ds * gi * (1.0 - gc ** 2),
            "f": ds * s_prev * gf * (1.0 - gf),
            "o": dht * tanh_s * go * (1.0 - go),
        }
        ds_next = ds * gf
        dh_next = sum(dpre[g] @ r64[g] for g in GATES)
        dx[t] = sum(dpre[g] @ w64[g] for g in GATES)
        xt = np.asarray(x[t], F64)
        for g in GATES:
            dw[g] += dpre[g].T @ xt
            dr[g] += dpre[g].T @ h_prev
            db[g] += dpre[g].sum(axis=0)
    f = lambda d: {g: v.astype(F32) for g, v in d.items()}  # noqa: E731
    return {"dx": dx.astype(F32), "dw": f(dw), "dr": f(dr), "db": f(db),
            "dh0": dh_next.astype(F32), "ds0": ds_next.astype(F32)}


# ---------------------------------------------------------------------------
# Convolution (reference cnn.py)
# ---------------------------------------------------------------------------
def conv_out_hw(h, w, r, s, stride, pad_h, pad_w):
    """Output extents (cnn.py:117-123)."""
    return (h + 2 * pad_h - r) // stride + 1, (w + 2 * pad_w - s) // stride + 1


def conv2d_forward_reference(i_nchw, w_kcrs, stride=1, pad_h=None, pad_w=None):
    """Direct convolution, float64, (r, s) loops + channel contraction (cnn.py:337-363).

    Same padding (R-1)/2 by default (cnn.py:79-87).
    """
    n, c, h, wd = i_nchw.shape
    k, _, r, s = w_kcrs.shape
    pad_h = (r - 1) // 2 if pad_h is None else pad_h
    pad_w = (s - 1) // 2 if pad_w is None else pad_w
    p, q = conv_out_hw(h, wd, r, s, stride, pad_h, pad_w)
    ipad = np.pad(np.asarray(i_nchw, F64), ((0, 0), (0, 0), (pad_h, pad_h), (pad_w, pad_w)))
    w64 = np.asarray(w_kcrs, F64)
    out = np.zeros((n, k, p, q))
    hs, ws = stride * (p - 1) + 1, stride * (q - 1) + 1
    for rr in range(r):
        for ss in range(s):
            win = ipad[:, :, rr: rr + hs: stride, ss: ss + ws: stride]
            out += np.einsum("nchw,kc->nkhw", win, w64[:, :, rr, ss], optimize=True)
    return out.astype(F32)


def conv2d_backward_data_reference(do_nkpq, w_kcrs, in_hw, stride=1, pad_h=None, pad_w=None):
    """dI for the forward above: scatter dO through the flipped stencil ("dual convolution",
    PAPER.md:281), float64, cropped to the unpadded input (no reference path; restated)."""
    n, k, p, q = do_nkpq.shape
    _, c, r, s = w_kcrs.shape
    h, wd = in_hw
    pad_h = (r - 1) // 2 if pad_h is None else pad_h
    pad_w = (s - 1) // 2 if pad_w is None else pad_w
    dpad = np.zeros((n, c, h + 2 * pad_h + stride, wd + 2 * pad_w + stride))
    do64 = np.asarray(do_nkpq, F64)
    w64 = np.asarray(w_kcrs, F64)
    hs, ws = stride * (p - 1) + 1, stride * (q - 1) + 1
    for rr in range(r):
        for ss in range(s):
            dpad[:, :, rr: rr + hs: stride, ss: ss + ws: stride] += np.einsum(
                "nkpq,kc->ncpq", do64, w64[:, :, rr, ss], optimize=True)
    return dpad[:, :, pad_h: pad_h + h, pad_w: pad_w + wd].astype(F32)


def conv2d_weight_update_reference(i_nchw, do_nkpq, r, s, stride=1, pad_h=None, pad_w=None):
    """dW[k][c][r][s] = sum_{n,p,q} dO[n][k][p][q] * I_pad[n][c][p*str+r][q*str+s] (restated)."""
    n, c, h, wd = i_nchw.shape
    _, k, p, q = do_nkpq.shape
    pad_h = (r - 1) // 2 if pad_h is None else pad_h
    pad_w = (s - 1) // 2 if pad_w is None else pad_w
    ipad = np.pad(np.asarray(i_nchw, F64), ((0, 0), (0, 0), (pad_h, pad_h), (pad_w, pad_w)))
    do64 = np.asarray(do_nkpq, F64)
    dw = np.zeros((k, c, r, s))
    hs, ws = stride * (p - 1) + 1, stride * (q - 1) + 1
    for rr in range(r):
        for ss in range(s):
            win = ipad[:, :, rr: rr + hs: stride, ss: ss + ws: stride]
            dw[:, :, rr, ss] = np.einsum("nkpq,ncpq->kc", do64, win, optimize=True)
    return dw.astype(F32)


# ResNet-50 conv table (reference bench.py:57-79): id, C, K, H, W, R, S, stride, count
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


def cpu_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
