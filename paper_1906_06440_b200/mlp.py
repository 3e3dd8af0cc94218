"""Multi-layer perceptron training step built from the FC passes (BASELINE config 2).

One step = for every layer the paper's three passes (fwd, bwd-data, weight
update) plus bias gradient and SGD, all on the BRGEMM engine:

    fwd   y_l  = relu(W_l y_{l-1} + b_l)                       (brk_fc_fwd)
    bwd   dz_L = dy * (y_L > 0), db_L, b_L -= lr db_L           (brk_fc_bias_grad)
          dz_{l-1} = (W_l^T dz_l) * (y_{l-1} > 0)               (brk_fc_bwd_data, mask fused)
          db_{l-1}, b_{l-1} -= lr db_{l-1}                      (brk_fc_bias_grad)
          dx = W_1^T dz_1                                       (brk_fc_bwd_data)
    upd   dW_l = dz_l y_{l-1}^T,  W_l -= lr dW_l                (brk_fc_upd, SGD fused)

Layouts are the reference's blocked FC layouts with b_n = b_c = b_k = 64
(activations [N_b][C_b][64][64], weights [K_b][C_b][64][64]); storage bf16,
accumulation fp32 in TMEM, weight/bias gradients fp32.  The whole step is a
fixed sequence of native launches on one stream, so it is captured once into
a CUDA graph and replayed.

Data parallel (``dist.py``): with a process group the per-layer dW/db are
all-reduced (NCCL) before the SGD apply, bucketed per layer in reverse order.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._device import require_cuda
from .fc import Activation, FcParams
from .tensor import BlockedTensor

B = 64


def flops_per_step(layers: int, n: int, c: int, k: int) -> int:
    """GEMM flops of fwd + bwd-data + upd over all layers: 3 * 2NCK per layer."""
    return layers * 3 * 2 * n * c * k


class MLP:
    """``layers`` x FC(width -> width) + ReLU on a minibatch of ``batch`` rows."""

    def __init__(self, layers: int = 4, width: int = 1024, batch: int = 2048, lr: float = 1e-3,
                 seed: int = 0, process_group=None, device: str = "cuda"):
        torch = require_cuda()
        if width % 128 or batch % 128:
            raise ValueError("MLP engine path needs width and batch multiples of 128")
        self.torch = torch
        self.L, self.C, self.N, self.lr = layers, width, batch, lr
        self.pg = process_group
        g = torch.Generator(device="cpu").manual_seed(seed)
        bf = torch.bfloat16
        cb = width // B
        nb = batch // B
        self._wbuf = [[], []]  # bf16 [Kb][Cb][64][64]; the fused step reads _wbuf[cur], writes _wbuf[1-cur]
        self._cur = 0
        self.bias = []   # fp32 [K]
        for _ in range(layers):
            w = (torch.rand(width, width, generator=g) * 2 - 1) / np.sqrt(width)
            self._wbuf[0].append(w.reshape(cb, B, cb, B).permute(0, 2, 3, 1).contiguous().to(device, bf))
            self.bias.append(((torch.rand(width, generator=g) * 2 - 1) * 0.1).to(device))
        if process_group is not None:
            # data parallel: every replica starts from rank 0's parameters (the ranks'
            # seeds may differ; only their data shards should)
            from .dist import broadcast_params

            broadcast_params(self._wbuf[0] + self.bias, process_group)
        # activations: y[0] is the input, y[l] the output of layer l
        self.y = [torch.empty(nb, cb, B, B, dtype=bf, device=device) for _ in range(layers + 1)]
        self.dz = [torch.empty(nb, cb, B, B, dtype=bf, device=device) for _ in range(layers + 1)]
        self.dy = torch.empty(nb, cb, B, B, dtype=bf, device=device)
        # all gradients in one flat fp32 buffer: one all-reduce bucket in data parallel
        self.grads = torch.empty(layers * (width * width + width), dtype=torch.float32, device=device)
        self.dw = [self.grads[l * width * width:(l + 1) * width * width].view(cb, cb, B, B) for l in range(layers)]
        off = layers * width * width
        self.db = [self.grads[off + l * width:off + (l + 1) * width] for l in range(layers)]
        lib = _lib.load()
        self.lib = lib
        self.ws = [torch.zeros(lib.brk_fc_bias_grad_workspace(width), dtype=torch.uint8, device=device)
                   for _ in range(layers)]
        # column-sum partials of dz_l (written by bwd-data of layer l+1, reduced by upd of layer l)
        self.colsum = [torch.zeros(batch // 32, width, dtype=torch.float32, device=device)
                       for _ in range(layers + 1)]
        upd_bytes = max(int(lib.brk_fc_upd_workspace(batch, width, width)), 16)
        self.upd_ws = [torch.zeros(upd_bytes, dtype=torch.uint8, device=device) for _ in range(layers)]
        self.graph = None
        self.launches_per_step = 0
        # whole-step persistent launch (brk_mlp_step): device pointer tables + dependency counters
        import ctypes
        import os

        self.fused = (os.environ.get("BRK_MLP_FUSED", "1") != "0" and layers <= 4
                      and width % 256 == 0 and batch % 256 == 0)
        # double-buffered weights: the weight update writes W - lr dW to the other buffer, so it
        # need not wait for the bwd-data pass that reads W (brk_mlp_step w_next)
        self._wbuf[1] = [w.clone() for w in self._wbuf[0]] if (self.fused and process_group is None) else self._wbuf[0]
        arr = lambda ts: (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])  # noqa: E731
        self._tables = [(arr(self.y), arr(self.dz), arr(self._wbuf[c]), arr(self._wbuf[1 - c]), arr(self.bias),
                         arr(self.dw), arr(self.db), arr(self.colsum)) for c in (0, 1)]
        self.graphs = None
        # dependency counters + split tickets (zeroed by every call) and parked half-accumulators
        self.step_ws = torch.zeros(max(int(lib.brk_mlp_step_workspace_bytes(layers, batch, width)), 16),
                                   dtype=torch.uint8, device=device)

    @property
    def w(self):
        """Current (latest) bf16 weights of every layer."""
        return self._wbuf[self._cur]

    # ------------------------------------------------------------------ params
    def params(self, l: int) -> FcParams:
        """Reference-API view of layer ``l`` (device bf16 weights)."""
        w = BlockedTensor(self.w[l], n_outer=2, logical_dims={"k": (0, 3), "c": (1, 2)})
        return FcParams(w=w, n=self.N, c=self.C, k=self.C, b_n=B, b_c=B, b_k=B,
                        activation=Activation.RELU, bias=self.bias[l])

    def load_input(self, x, dy) -> None:
        """Copy a step's input and output-gradient (blocked, bf16) into the static buffers."""
        self.y[0].copy_(x, non_blocking=True)
        self.dy.copy_(dy, non_blocking=True)

    # ------------------------------------------------------------------ passes
    def _check(self, rc):
        _lib.check(rc, RuntimeError)

    def forward(self, stream: int) -> int:
        lib, n, c = self.lib, self.N, self.C
        for l in range(self.L):
            self._check(lib.brk_fc_fwd(self.y[l].data_ptr(), self.w[l].data_ptr(), self.bias[l].data_ptr(),
                                       self.y[l + 1].data_ptr(), n, c, c, B, B, B, 1, _lib.BRK_BF16, stream))
        return self.L

    def backward_update(self, stream: int, apply_sgd: bool = True, reducer=None) -> int:
        """bwd-data + bias grad + weight update for all layers; returns launches issued.

        With a ``reducer`` (data parallel) each layer's (dW, db) all-reduce is
        submitted on the communication stream right after its weight update,
        overlapping the remaining backward passes.
        """
        lib, n, c, L = self.lib, self.N, self.C, self.L
        lr = self.lr if apply_sgd else 0.0
        launches = 0
        # top layer: dz_L = dy * (y_L > 0); db_L (+ bias SGD)
        self._check(lib.brk_fc_bias_grad(self.dy.data_ptr(), self.y[L].data_ptr(), self.dz[L].data_ptr(),
                                         self.db[L - 1].data_ptr(), self.ws[L - 1].data_ptr(), n, c, B, B,
                                         self.bias[L - 1].data_ptr() if apply_sgd else None, lr, stream))
        launches += 1
        for l in range(L, 0, -1):
            # bwd-data first (it reads W_l before the fused SGD rewrites it); its epilogue
            # applies layer l-1's ReLU mask and writes column-sum partials of dz_{l-1}
            mask = self.y[l - 1].data_ptr() if l > 1 else None
            colsum = self.colsum[l - 1].data_ptr() if l > 1 else None
            self._check(lib.brk_fc_bwd_data(self.dz[l].data_ptr(), self.w[l - 1].data_ptr(), mask,
                                            self.dz[l - 1].data_ptr(), colsum, n, c, c, B, B, B,
                                            _lib.BRK_BF16, stream))
            launches += 1
            # weight update (+ SGD); for l < L it also reduces dz_l's column sums into db_l (+ bias SGD)
            parts = self.colsum[l].data_ptr() if l < L else None
            self._check(lib.brk_fc_upd(self.y[l - 1].data_ptr(), self.dz[l].data_ptr(), self.dw[l - 1].data_ptr(),
                                       self.w[l - 1].data_ptr() if apply_sgd else None, lr,
                                       parts, n // 32, self.db[l - 1].data_ptr() if parts else None,
                                       self.bias[l - 1].data_ptr() if (parts and apply_sgd) else None, lr,
                                       self.upd_ws[l - 1].data_ptr(), self.upd_ws[l - 1].numel(),
                                       n, c, c, B, B, B, _lib.BRK_BF16, stream))
            launches += 1
            if reducer is not None:
                reducer.submit([self.dw[l - 1], self.db[l - 1]])
        return launches

    def fused_step(self, stream: int) -> int:
        """The whole step as ONE persistent engine launch (brk_mlp_step): 3L
        dependent GEMM problems with tile-level dependency counters."""
        y, dz, w, w_next, b, dw, db, cs = self._tables[self._cur]
        self._check(self.lib.brk_mlp_step(self.L, self.N, self.C, y, dz, self.dy.data_ptr(), w, w_next, b, dw, db,
                                          cs, self.lr, self.step_ws.data_ptr(), self.step_ws.numel(),
                                          stream))
        self._cur ^= 1
        return 1

    def step(self, stream: int | None = None) -> int:
        """One fwd/bwd/upd step on the current buffers (single GPU: SGD fused)."""
        torch = self.torch
        s = torch.cuda.current_stream().cuda_stream if stream is None else stream
        if self.pg is None and self.fused:
            n = self.fused_step(s)
        elif self.fused:
            # data parallel: gradients from the fused step (no SGD), one all-reduce bucket, SGD apply
            y, dz, w, _, b, dw, db, cs = self._tables[self._cur]
            self._check(self.lib.brk_mlp_step(self.L, self.N, self.C, y, dz, self.dy.data_ptr(), w, None, b, dw, db,
                                              cs, 0.0, self.step_ws.data_ptr(), self.step_ws.numel(), s))
            self._reducer().submit([self.grads])
            n = 1 + self._allreduce_apply(s)
        elif self.pg is None:
            n = self.forward(s) + self.backward_update(s, apply_sgd=True)
        else:
            n = self.forward(s) + self.backward_update(s, apply_sgd=False, reducer=self._reducer())
            n += self._allreduce_apply(s)
        self.launches_per_step = n
        return n

    def _reducer(self):
        if getattr(self, "_grad_reducer", None) is None:
            from .dist import GradientReducer

            self._grad_reducer = GradientReducer(group=self.pg)
        return self._grad_reducer

    def _allreduce_apply(self, stream: int) -> int:
        """DP exchange: wait for the per-layer all-reduces (sum), then SGD with lr / world."""
        from .dist import sgd_scale

        red = self._reducer()
        red.wait()
        scale = sgd_scale(self.lr, red.world)
        launches = 0
        for l in range(self.L - 1, -1, -1):
            self._check(self.lib.brk_sgd_apply(self.w[l].data_ptr(), self.dw[l].data_ptr(), scale,
                                               self.dw[l].numel(), _lib.BRK_BF16, stream))
            self._check(self.lib.brk_sgd_apply(self.bias[l].data_ptr(), self.db[l].data_ptr(), scale,
                                               self.db[l].numel(), _lib.BRK_F32, stream))
            launches += 2
        return launches

    # ------------------------------------------------------------------ graphs
    def capture(self):
        """Capture one single-GPU step into a CUDA graph (replay with ``replay``)."""
        torch = self.torch
        if self.pg is not None:
            raise RuntimeError("graph capture is for the single-GPU step; DP steps call step()")
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.step(side.cuda_stream)  # warm: encodes tensor maps, sets smem attributes
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        # one graph per weight-buffer parity (the fused step alternates the buffers)
        self.graphs = {}
        for _ in range(2 if self.fused else 1):
            g = torch.cuda.CUDAGraph()
            cur = self._cur
            with torch.cuda.graph(g, stream=side):
                self.step(side.cuda_stream)
            self._cur = cur
            self.graphs[cur] = g
            if self.fused:
                self._cur ^= 1
        self.graph = self.graphs[self._cur]
        return self.graph

    def replay(self):
        self.graphs[self._cur].replay()
        if self.fused:
            self._cur ^= 1

    def train_step(self, x_host, dy_host, out_host=None):
        """Public end-to-end step: H2D of the step's input and output gradient
        (pinned host, blocked bf16), the fwd/bwd/upd step (graph replay when
        captured), and a D2H read of the step's result (the last layer's bias
        gradient) into ``out_host``.  Returns ``out_host``."""
        torch = self.torch
        self.y[0].copy_(x_host, non_blocking=True)
        self.dy.copy_(dy_host, non_blocking=True)
        if self.graph is not None:
            self.replay()
        else:
            self.step()
        if out_host is None:
            out_host = torch.empty(self.C, dtype=torch.float32, pin_memory=True)
        out_host.copy_(self.db[self.L - 1], non_blocking=True)
        return out_host

    def train(self, xs, dys, outs):
        """Pipelined end-to-end training over len(xs) steps through the public API:
        every step's input and output gradient are copied from pinned host memory
        (on a copy stream, into a double-buffered device staging area, overlapping
        the previous step's compute), the step runs (graph replay when captured) and
        its result (the last layer's bias gradient) is read back into ``outs[i]``."""
        torch = self.torch
        n = len(xs)
        main = torch.cuda.current_stream()
        copy = getattr(self, "_copy_stream", None) or torch.cuda.Stream()
        self._copy_stream = copy
        if getattr(self, "_staging", None) is None:
            self._staging = [(torch.empty_like(self.y[0]), torch.empty_like(self.dy)) for _ in range(2)]
        copied = [torch.cuda.Event() for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        copy.wait_stream(main)

        def h2d(i):
            sx, sdy = self._staging[i % 2]
            with torch.cuda.stream(copy):
                if i >= 2:
                    copy.wait_event(free[i % 2])
                sx.copy_(xs[i], non_blocking=True)
                sdy.copy_(dys[i], non_blocking=True)
                copied[i % 2].record(copy)

        h2d(0)
        for i in range(n):
            if i + 1 < n:
                h2d(i + 1)
            main.wait_event(copied[i % 2])
            sx, sdy = self._staging[i % 2]
            self.y[0].copy_(sx, non_blocking=True)
            self.dy.copy_(sdy, non_blocking=True)
            free[i % 2].record(main)
            if self.graph is not None:
                self.replay()
            else:
                self.step()
            outs[i].copy_(self.db[self.L - 1], non_blocking=True)
        return outs


class MlpTF32:
    """The same MLP training step with the reference's own fp32 storage and TF32
    tensor-core math (north_star "bf16 and TF32 inputs"): activations, weights
    and gradients fp32 in HBM.  By default the whole step is ONE persistent launch
    of the fused step kernel in its TF32 variant (``brk_mlp_step_dt`` with
    BRK_F32: kind::tf32 MMAs on 32-element fp32 atoms, fp32 epilogues in 32-column
    TMA boxes, double-buffered weights).  ``BRK_MLP_FUSED=0`` runs the per-pass
    path, every GEMM on the engine's TF32 path, 4L + 1 + L native launches:

        fwd   y_l = relu(W_l y_{l-1} + b_l)                 brk_fc_fwd(F32)
        top   dz_L = dy * (y_L > 0), db_L, b_L -= lr db_L    brk_fc_bias_grad_dt(F32)
        bwd   dz_{l-1} = (W_l^T dz_l) * (y_{l-1} > 0)        brk_fc_bwd_data(F32, mask, column sums)
        upd   dW_l = dz_l y_{l-1}^T, db_{l-1} (+ bias SGD)   brk_fc_upd(F32)
        sgd   W_l -= lr dW_l                                 brk_sgd_apply(F32)

    (the fused-SGD epilogue writes bf16 weights, so fp32 weights take the separate apply)."""

    def __init__(self, layers: int = 4, width: int = 1024, batch: int = 2048, lr: float = 1e-3,
                 seed: int = 0, device: str = "cuda"):
        torch = require_cuda()
        if width % 128 or batch % 256:
            raise ValueError("TF32 MLP engine path needs width % 128 == 0 and batch % 256 == 0")
        self.torch = torch
        self.L, self.C, self.N, self.lr = layers, width, batch, lr
        g = torch.Generator(device="cpu").manual_seed(seed)
        cb, nb = width // B, batch // B
        f32 = torch.float32
        self.w, self.bias = [], []
        for _ in range(layers):
            w = (torch.rand(width, width, generator=g) * 2 - 1) / np.sqrt(width)
            self.w.append(w.reshape(cb, B, cb, B).permute(0, 2, 3, 1).contiguous().to(device))
            self.bias.append(((torch.rand(width, generator=g) * 2 - 1) * 0.1).to(device))
        self.y = [torch.empty(nb, cb, B, B, dtype=f32, device=device) for _ in range(layers + 1)]
        self.dz = [torch.empty(nb, cb, B, B, dtype=f32, device=device) for _ in range(layers + 1)]
        self.dy = torch.empty(nb, cb, B, B, dtype=f32, device=device)
        self.dw = [torch.empty(cb, cb, B, B, dtype=f32, device=device) for _ in range(layers)]
        self.db = [torch.empty(width, dtype=f32, device=device) for _ in range(layers)]
        self.colsum = [torch.zeros(batch // 32, width, dtype=f32, device=device) for _ in range(layers + 1)]
        lib = _lib.load()
        self.lib = lib
        self.ws_top = torch.zeros(lib.brk_fc_bias_grad_workspace(width), dtype=torch.uint8, device=device)
        upd_bytes = max(int(lib.brk_fc_upd_workspace(batch, width, width)), 16)
        self.upd_ws = [torch.zeros(upd_bytes, dtype=torch.uint8, device=device) for _ in range(layers)]
        self.launches_per_step = 0
        import ctypes
        import os

        self.fused = (os.environ.get("BRK_MLP_FUSED", "1") != "0" and layers <= 4
                      and width % 256 == 0 and batch % 256 == 0)
        if self.fused:
            # double-buffered weights (the step writes W - lr dW to the other buffer)
            self._wbuf = [self.w, [w.clone() for w in self.w]]
            self._cur = 0
            arr = lambda ts: (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])  # noqa: E731
            self._tables = [(arr(self.y), arr(self.dz), arr(self._wbuf[c]), arr(self._wbuf[1 - c]), arr(self.bias),
                             arr(self.dw), arr(self.db), arr(self.colsum)) for c in (0, 1)]
            self.step_ws = torch.zeros(max(int(lib.brk_mlp_step_workspace_bytes(layers, batch, width)), 16),
                                       dtype=torch.uint8, device=device)

    def load_input(self, x, dy) -> None:
        self.y[0].copy_(x, non_blocking=True)
        self.dy.copy_(dy, non_blocking=True)

    def step(self, stream: int | None = None) -> int:
        torch, lib, n, c, L, lr = self.torch, self.lib, self.N, self.C, self.L, self.lr
        s = torch.cuda.current_stream().cuda_stream if stream is None else stream
        F = _lib.BRK_F32
        if self.fused:
            y, dz, w, w_next, b, dw, db, cs = self._tables[self._cur]
            _lib.check(lib.brk_mlp_step_dt(L, n, c, y, dz, self.dy.data_ptr(), w, w_next, b, dw, db, cs, lr,
                                           self.step_ws.data_ptr(), self.step_ws.numel(), F, s), RuntimeError)
            self._cur ^= 1
            self.w = self._wbuf[self._cur]
            self.launches_per_step = 1
            return 1
        chk = lambda rc: _lib.check(rc, RuntimeError)  # noqa: E731
        for l in range(L):
            chk(lib.brk_fc_fwd(self.y[l].data_ptr(), self.w[l].data_ptr(), self.bias[l].data_ptr(),
                               self.y[l + 1].data_ptr(), n, c, c, B, B, B, 1, F, s))
        chk(lib.brk_fc_bias_grad_dt(self.dy.data_ptr(), self.y[L].data_ptr(), self.dz[L].data_ptr(),
                                    self.db[L - 1].data_ptr(), self.ws_top.data_ptr(), n, c, B, B,
                                    self.bias[L - 1].data_ptr(), lr, F, s))
        launches = L + 1
        for l in range(L, 0, -1):
            mask = self.y[l - 1].data_ptr() if l > 1 else None
            colsum = self.colsum[l - 1].data_ptr() if l > 1 else None
            chk(lib.brk_fc_bwd_data(self.dz[l].data_ptr(), self.w[l - 1].data_ptr(), mask,
                                    self.dz[l - 1].data_ptr(), colsum, n, c, c, B, B, B, F, s))
            parts = self.colsum[l].data_ptr() if l < L else None
            chk(lib.brk_fc_upd(self.y[l - 1].data_ptr(), self.dz[l].data_ptr(), self.dw[l - 1].data_ptr(),
                               None, 0.0, parts, n // 32, self.db[l - 1].data_ptr() if parts else None,
                               self.bias[l - 1].data_ptr() if parts else None, lr,
                               self.upd_ws[l - 1].data_ptr(), self.upd_ws[l - 1].numel(),
                               n, c, c, B, B, B, F, s))
            chk(lib.brk_sgd_apply(self.w[l - 1].data_ptr(), self.dw[l - 1].data_ptr(), lr,
                                  self.dw[l - 1].numel(), F, s))
            launches += 3
        self.launches_per_step = launches
        return launches
