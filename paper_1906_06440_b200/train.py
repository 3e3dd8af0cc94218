"""Data-parallel training steps for the conv and LSTM workloads,
beside the MLP step in ``mlp.py``.  One process per GPU; the minibatch is
sharded, fwd and bwd-data need no communication, and the single exchange is
the weight-gradient sum after each weight-update pass (NCCL all-reduce on a
communication stream, ``dist.GradientReducer``), issued per layer in reverse
layer order so it overlaps the backward passes still to run, then SGD with
lr / world (``dist.sgd_scale``).  Initial weights are broadcast from rank 0.

* ``ResNetConvs`` — the 53 convolutions of ResNet-50 (the reference bench
  table, 20 shapes x occurrence count, /root/reference/pkg/src/brkernels/
  bench.py:57-79), each an independent blocked conv layer with its own
  weights, at a global minibatch of N images split contiguously over the
  ranks (the reference's minibatch-first strategy, cnn.py:158-176): strong
  scaling.  Layers 2-20 call the implicit-GEMM engine through the C-ABI with
  preallocated buffers; the 3-channel stem goes through the public
  conv2d_* API (im2col + dense engine GEMM).
* ``LstmDP`` — the LSTM cell at N sequences PER RANK (weak scaling, SURVEY
  8e): fwd + BPTT on the rank's sequences; dW, dR, db all-reduced as each
  weight-gradient GEMM is issued, overlapping the remaining BPTT products.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._device import require_cuda
from .cnn import ConvSpec, conv2d_backward_data, conv2d_forward, conv2d_weight_update
from .dist import GradientReducer, broadcast_params, sgd_scale, shard_range
from .tensor import BlockedTensor

# (id, C, K, H, W, R, S, stride, count) — reference bench.py:57-79
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


def _world_rank(pg):
    if pg is None:
        return 1, 0
    import torch.distributed as dist

    return dist.get_world_size(pg), dist.get_rank(pg)


def conv_flops(spec: ConvSpec) -> float:
    """2 N K C R S P Q (reference bench.py flops_conv)."""
    return 2.0 * spec.n * spec.k * spec.c * spec.r * spec.s * spec.out_h * spec.out_w


class _ConvLayer:
    """One conv instance: bf16 blocked weights (own), fp32 dW, shared activation buffers."""

    def __init__(self, spec: ConvSpec, w, bufs):
        self.spec, self.w, self.bufs = spec, w, bufs
        torch = require_cuda()
        self.dw = torch.empty(w.shape, dtype=torch.float32, device="cuda")


class ResNetConvs:
    """ResNet-50's 53 convolutions as one data-parallel training step (strong scaling)."""

    def __init__(self, n_global: int = 256, layers=None, lr: float = 1e-3, seed: int = 0,
                 process_group=None, counts: bool = True):
        torch = require_cuda()
        self.pg = process_group
        self.world, self.rank = _world_rank(process_group)
        shard = shard_range(n_global, self.rank, self.world)
        self.n_global, self.n_local, self.lr = n_global, len(shard), lr
        if self.n_local < 1:
            raise ValueError(f"minibatch {n_global} leaves rank {self.rank} of {self.world} without images")
        self.lib = _lib.load()
        g = torch.Generator(device="cuda").manual_seed(seed)
        gd = torch.Generator(device="cuda").manual_seed(1000 + seed * 997 + self.rank)  # data differs per rank
        self.layers: list[_ConvLayer] = []
        self.shapes = []
        n = self.n_local
        for lid, c, k, h, w, r, s, st, cnt in RESNET50_ROWS:
            if layers is not None and lid not in layers:
                continue
            spec = ConvSpec(n=n, c=c, k=k, h=h, w=w, r=r, s=s, stride=st)
            bc, bk = spec.b_c, spec.b_k
            bufs = {
                "x": (torch.rand((n, c // bc, h, w, bc), generator=gd, device="cuda") * 2 - 1).bfloat16(),
                "dout": (torch.rand((n, k // bk, spec.out_h, spec.out_w, bk), generator=gd, device="cuda") * 2
                         - 1).bfloat16(),
                "out": torch.empty((n, k // bk, spec.out_h, spec.out_w, bk), dtype=torch.bfloat16, device="cuda"),
                "din": torch.empty((n, c // bc, h, w, bc), dtype=torch.bfloat16, device="cuda"),
            }
            nb = self.lib.brk_conv_upd_workspace(*self._geom(spec)) if bc == 64 and bk == 64 else 0
            bufs["ws"] = torch.empty(max(int(nb), 16), dtype=torch.uint8, device="cuda")
            bufs["ws_bytes"] = int(nb)
            self.shapes.append((lid, spec, cnt if counts else 1))
            for _ in range(cnt if counts else 1):
                wt = ((torch.rand((k // bk, c // bc, r, s, bc, bk), generator=g, device="cuda") * 2 - 1)
                      / np.sqrt(c * r * s)).bfloat16()
                self.layers.append(_ConvLayer(spec, wt, bufs))
        if process_group is not None:
            broadcast_params([lay.w for lay in self.layers], process_group)
        self.reducer = GradientReducer(group=process_group) if process_group is not None else None

    @staticmethod
    def _geom(spec):
        return (spec.n, spec.c, spec.k, spec.h, spec.w, spec.r, spec.s, spec.stride, spec.pad_h, spec.pad_w)

    def flops_per_step(self, local: bool = True) -> float:
        """fwd + bwd-data + upd GEMM flops of every conv (stem bwd-data included)."""
        n = self.n_local if local else self.n_global
        return sum(3.0 * conv_flops(lay.spec) * n / lay.spec.n for lay in self.layers)

    def _engine(self, spec):
        return spec.b_c == 64 and spec.b_k == 64

    def _fwd(self, lay, sp):
        spec, b = lay.spec, lay.bufs
        if self._engine(spec):
            _lib.check(self.lib.brk_conv_fwd(b["x"].data_ptr(), lay.w.data_ptr(), None, b["out"].data_ptr(),
                                             *self._geom(spec), 64, 64, 0, _lib.BRK_BF16, sp))
            return 1
        xi = BlockedTensor(b["x"], 4, {"n": 0, "c": (1, 4), "h": 2, "w": 3})
        wi = BlockedTensor(lay.w, 4, {"k": (0, 5), "c": (1, 4), "r": 2, "s": 3})
        b["out"].copy_(conv2d_forward(spec, xi, wi).data)
        return 2

    def _bwd_upd(self, lay, sp):
        spec, b = lay.spec, lay.bufs
        if self._engine(spec):
            _lib.check(self.lib.brk_conv_bwd_data(b["dout"].data_ptr(), lay.w.data_ptr(), b["din"].data_ptr(),
                                                  *self._geom(spec), 64, 64, _lib.BRK_BF16, sp))
            _lib.check(self.lib.brk_conv_upd(b["x"].data_ptr(), b["dout"].data_ptr(), lay.dw.data_ptr(), None, 0.0,
                                             b["ws"].data_ptr() if b["ws_bytes"] else None, b["ws_bytes"],
                                             *self._geom(spec), 64, 64, _lib.BRK_BF16, sp))
            return 2
        xi = BlockedTensor(b["x"], 4, {"n": 0, "c": (1, 4), "h": 2, "w": 3})
        wi = BlockedTensor(lay.w, 4, {"k": (0, 5), "c": (1, 4), "r": 2, "s": 3})
        do = BlockedTensor(b["dout"], 4, {"n": 0, "k": (1, 4), "p": 2, "q": 3})
        b["din"].copy_(conv2d_backward_data(spec, do, wi).data)
        lay.dw.copy_(conv2d_weight_update(spec, xi, do).data)
        return 5

    def step(self) -> int:
        """fwd of every conv, then (reverse order) bwd-data + weight update with the dW
        all-reduce submitted per layer, then SGD.  Returns the native launches issued."""
        torch = require_cuda()
        sp = torch.cuda.current_stream().cuda_stream
        launches = 0
        for lay in self.layers:
            launches += self._fwd(lay, sp)
        for lay in reversed(self.layers):
            launches += self._bwd_upd(lay, sp)
            if self.reducer is not None:
                self.reducer.submit([lay.dw])
        if self.reducer is not None:
            self.reducer.wait()
        scale = sgd_scale(self.lr, self.world)
        for lay in self.layers:
            _lib.check(self.lib.brk_sgd_apply(lay.w.data_ptr(), lay.dw.data_ptr(), scale, lay.w.numel(),
                                              _lib.BRK_BF16, sp))
            launches += 1
        return launches


def _cat_of(parts):
    """The gate-concatenated buffer that ``parts`` (consecutive row slices) were cut from,
    or a concatenation when they are not such slices."""
    base = parts[0]._base
    if (base is not None and base.is_contiguous() and all(t._base is base for t in parts)
            and parts[0].data_ptr() == base.data_ptr() and base.numel() == sum(t.numel() for t in parts)
            and all(parts[i + 1].data_ptr() == parts[i].data_ptr() + parts[i].numel() * parts[i].element_size()
                    for i in range(len(parts) - 1))):
        return base.reshape(-1, *parts[0].shape[1:]) if parts[0].dim() > 1 else base.reshape(-1)
    import torch

    return torch.cat(parts)


class LstmDP:
    """LSTM cell training step, data parallel over sequences (weak scaling: N per rank)."""

    def __init__(self, t_steps: int = 50, n_local: int = 168, c: int = 1024, k: int = 1024, lr: float = 1e-3,
                 seed: int = 0, process_group=None, precision: str = "bf16"):
        torch = require_cuda()
        from .lstm import GATE_NAMES, LstmCellWeights, LstmParams

        self.pg = process_group
        self.world, self.rank = _world_rank(process_group)
        self.lr, self.precision = lr, precision
        self.T, self.N, self.C, self.K = t_steps, n_local, c, k
        wt = LstmCellWeights.random(np.random.default_rng([seed, 303]), c, k)
        params = LstmParams.from_dense(wt, t_steps, n_local)
        # fp32 master weights, dense and gate-concatenated as the BPTT gradients come out of
        # lstm_backward (dW_cat [4K][C], dR_cat [4K][K], db_cat [4K]); the params' blocked
        # W_g [K_b][C_b][b_c][b_k] / R_g and bias_g are strided views into them, so the public
        # params always hold the current weights and SGD is three contiguous updates
        self.w32 = torch.from_numpy(np.concatenate([getattr(wt, f"w_{g}") for g in GATE_NAMES])).cuda().float()
        self.r32 = torch.from_numpy(np.concatenate([getattr(wt, f"r_{g}") for g in GATE_NAMES])).cuda().float()
        self.b32 = torch.from_numpy(np.concatenate([np.asarray(getattr(wt, f"bias_{g}"), np.float32).reshape(-1)
                                                    for g in GATE_NAMES])).cuda()
        if process_group is not None:
            broadcast_params([self.w32, self.r32, self.b32], process_group)
        for i, g in enumerate(GATE_NAMES):
            getattr(params, f"w_{g}").data = self._blocked(self.w32, i, c, params.b_c, params.b_k)
            getattr(params, f"r_{g}").data = self._blocked(self.r32, i, k, params.b_k, params.b_k)
            setattr(params, f"bias_{g}", self.b32[i * k:(i + 1) * k])
        self.params = params
        self.gates = GATE_NAMES
        rng = np.random.default_rng([seed, 303, 1 + self.rank])  # data differs per rank
        self.x = torch.from_numpy(rng.uniform(-1, 1, (t_steps, n_local, c)).astype(np.float32)).cuda()
        self.dh = torch.from_numpy(rng.uniform(-1, 1, (t_steps, n_local, k)).astype(np.float32)).cuda()
        self.reducer = GradientReducer(group=process_group) if process_group is not None else None

    def _blocked(self, master, gate, cols, bx, bk):
        """W_g (K, X) rows gate*K.. of a dense master as the blocked [K_b][X_b][b_x][b_k] view."""
        k = self.K
        return master[gate * k:(gate + 1) * k].view(k // bk, bk, cols // bx, bx).permute(0, 2, 3, 1)

    def _refresh_device_copies(self):
        """Rebuild the kernels' operand copies straight from the updated masters (lstm._DeviceCell /
        _SeqCell) and key them on the params as they are now, so the next lstm_forward does not
        rebuild them through the per-gate blocked views: one cast per bf16 operand, one
        transposing cast for R^T, one copy per blocked fp32 stack (per-step TF32 kernels)."""
        from .lstm import _DeviceCell, _params_key, _SeqCell

        torch = require_cuda()
        p, k, c = self.params, self.K, self.C
        dc = _DeviceCell.__new__(_DeviceCell)
        dc.W = self.w32.view(4, k // p.b_k, p.b_k, c // p.b_c, p.b_c).permute(0, 1, 3, 4, 2).contiguous()
        dc.R = self.r32.view(4, k // p.b_k, p.b_k, k // p.b_k, p.b_k).permute(0, 1, 3, 4, 2).contiguous()
        dc.bias = self.b32
        sc = _SeqCell.__new__(_SeqCell)
        sc.w_cat = self.w32.to(torch.bfloat16)
        sc.r_cat = self.r32.to(torch.bfloat16)
        sc.rt_cat = torch.empty((4 * k, k), dtype=torch.bfloat16, device="cuda")
        sc.rt_cat.view(4, k, k).copy_(self.r32.view(4, k, k).transpose(1, 2))
        sc.bias = self.b32
        object.__setattr__(p, "_brk_device_cell", (_params_key(p), dc))
        object.__setattr__(p, "_brk_seq_cell", sc)

    def flops_per_step(self) -> float:
        """fwd 2TN(4KC + 4KK), bwd + upd twice that (reference bench.py flops_lstm_fwd)."""
        return 3 * 2.0 * self.T * self.N * (4 * self.K * self.C + 4 * self.K * self.K)

    def step(self):
        from . import precision as prec_ctx
        from .lstm import lstm_backward, lstm_forward

        p = self.params
        with prec_ctx(self.precision):
            seq = lstm_forward(p, self.x)
            grads = lstm_backward(p, self.x, seq, self.dh, reducer=self.reducer)
        if self.reducer is not None:
            self.reducer.wait()
        scale = sgd_scale(self.lr, self.world)
        torch = require_cuda()
        dw, dr, db = (_cat_of([getattr(grads, f)[g] for g in self.gates]) for f in ("dw", "dr", "db"))
        torch._foreach_add_([self.w32, self.r32, self.b32], [dw, dr, db], alpha=-scale)
        self._refresh_device_copies()
        return grads
