"""The reference package's fp64 oracle functions, under their reference names
(``brkernels.__init__``, reference ``__init__.py:3-54``): ``brgemm_reference``,
``fc_forward_reference``, ``lstm_forward_reference``, ``conv2d_forward_reference``.

These are the reference API's COMPARISON TARGETS, kept so that a caller doing
``bk.brgemm_reference(...)`` keeps working after switching packages.  They
are host NumPy (float64 accumulation, one float32 rounding of each stored
value, the reference's semantics) and are OFF every compute path: nothing in
this package calls them, and the GPU entry points never fall back to them.
The test-side checker (``oracle/brk_oracle.py``) is a separate restatement;
the two are checked against each other and against the reference's own
golden vectors in tests/test_reference_api.py.
"""

from __future__ import annotations

import numpy as np

from .brgemm import BrgemmSpec, _check_blocks
from .fc import Activation
from .lstm import GATE_NAMES, LstmCellWeights, LstmStateSequence
from .tensor import FP32, LayoutError


def brgemm_reference(a_blocks, b_blocks, c, spec: BrgemmSpec) -> np.ndarray:
    """C = alpha * sum_i B_i @ A_i + beta * C in float64, one f32 round, in place (brgemm.py:210-225)."""
    _check_blocks(a_blocks, b_blocks, c, spec)
    total = np.zeros(np.shape(c), dtype=np.float64)
    if spec.alpha != 0.0:
        for a, b in zip(a_blocks, b_blocks):
            total += np.matmul(np.asarray(b, np.float64), np.asarray(a, np.float64))
        total *= spec.alpha
    if spec.beta != 0.0:
        total += spec.beta * np.asarray(c, np.float64)
    c[...] = total
    return c


def fc_forward_reference(w_dense, x_dense, activation: Activation = Activation.IDENTITY) -> np.ndarray:
    """Y = g(W @ X), W (K, C), X (C, N), float64 accumulation (fc.py:166-179)."""
    w_dense = np.asarray(w_dense)
    x_dense = np.asarray(x_dense)
    if w_dense.ndim != 2 or x_dense.ndim != 2 or w_dense.shape[1] != x_dense.shape[0]:
        raise LayoutError(f"shape mismatch: W {w_dense.shape} X {x_dense.shape}")
    z = w_dense.astype(np.float64) @ x_dense.astype(np.float64)
    if activation is Activation.RELU:
        z = np.maximum(z, 0.0)
    elif activation is Activation.SIGMOID:
        z = 1.0 / (1.0 + np.exp(-z))
    return z.astype(FP32)


def lstm_forward_reference(weights: LstmCellWeights, x, h_init=None, s_init=None,
                           keep_gates: bool = False) -> LstmStateSequence:
    """Whole-matrix LSTM oracle: float64 within a step, f32 h/s handed between steps (lstm.py:330-378)."""
    weights.validate()
    k, c = weights.w_i.shape
    x = np.asarray(x)
    t_steps, n = x.shape[0], x.shape[1]
    if x.shape != (t_steps, n, c):
        raise LayoutError(f"x has shape {x.shape}, expected (T, N, {c})")
    x64 = x.astype(np.float64)
    h_prev = np.zeros((n, k)) if h_init is None else np.asarray(h_init, np.float64)
    s_prev = np.zeros((n, k)) if s_init is None else np.asarray(s_init, np.float64)
    w64 = {g: np.asarray(getattr(weights, f"w_{g}"), np.float64) for g in GATE_NAMES}
    r64 = {g: np.asarray(getattr(weights, f"r_{g}"), np.float64) for g in GATE_NAMES}
    b64 = {g: np.asarray(getattr(weights, f"bias_{g}"), np.float64) for g in GATE_NAMES}
    h = np.empty((t_steps, n, k), FP32)
    s = np.empty((t_steps, n, k), FP32)
    gates = {g: np.empty((t_steps, n, k), FP32) for g in GATE_NAMES} if keep_gates else None
    for t in range(t_steps):
        pre = {g: x64[t] @ w64[g].T + h_prev @ r64[g].T + b64[g] for g in GATE_NAMES}
        act = {"i": 1.0 / (1.0 + np.exp(-pre["i"])), "c": np.tanh(pre["c"]),
               "f": 1.0 / (1.0 + np.exp(-pre["f"])), "o": 1.0 / (1.0 + np.exp(-pre["o"]))}
        s_t = act["f"] * s_prev + act["i"] * act["c"]
        h[t] = act["o"] * np.tanh(s_t)
        s[t] = s_t
        if gates is not None:
            for g in GATE_NAMES:
                gates[g][t] = act[g]
        h_prev = h[t].astype(np.float64)
        s_prev = s[t].astype(np.float64)
    return LstmStateSequence(h=h, s=s, gates=gates)


def conv2d_forward_reference(spec, i_nchw, w_kcrs) -> np.ndarray:
    """Direct (r, s)-loop convolution over NCHW / KCRS in float64 (cnn.py:337-363)."""
    i_nchw = np.asarray(i_nchw)
    w_kcrs = np.asarray(w_kcrs)
    if i_nchw.shape != (spec.n, spec.c, spec.h, spec.w):
        raise LayoutError(f"input shape {i_nchw.shape} does not match spec")
    if w_kcrs.shape != (spec.k, spec.c, spec.r, spec.s):
        raise LayoutError(f"weight shape {w_kcrs.shape} does not match spec")
    p, q, st = spec.out_h, spec.out_w, spec.stride
    i64 = np.pad(i_nchw.astype(np.float64),
                 ((0, 0), (0, 0), (spec.pad_h, spec.pad_h), (spec.pad_w, spec.pad_w)))
    w64 = w_kcrs.astype(np.float64)
    out = np.zeros((spec.n, spec.k, p, q))
    hs, ws = st * (p - 1) + 1, st * (q - 1) + 1
    for r in range(spec.r):
        for s in range(spec.s):
            win = i64[:, :, r:r + hs:st, s:s + ws:st]  # (n, c, p, q)
            out += np.einsum("ncpq,kc->nkpq", win, w64[:, :, r, s], optimize=True)
    return out.astype(FP32)


__all__ = ["brgemm_reference", "conv2d_forward_reference", "fc_forward_reference", "lstm_forward_reference"]
