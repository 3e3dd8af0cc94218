"""Data parallelism over the minibatch: one process per GPU.

The paper's primitives shard naturally over the minibatch (conv: images,
FC: N_b row blocks, LSTM: sequences).  Forward and backward-data need no
communication; the single exchange step is the weight-gradient sum after
each weight-update pass:

    dW_total = sum_ranks dW_rank        (all-reduce, NCCL over NVLink/NVSwitch)
    W -= (lr / world) * dW_total        (SGD with the global-mean gradient)

Gradients are bucketed per layer and reduced in reverse layer order on a
dedicated communication stream, so the all-reduce of layer l overlaps the
backward passes of layers l-1 .. 1 (``GradientReducer``).  The same code runs
over gloo on CPU tensors (tests) and NCCL on CUDA tensors (bench.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .partition import split_evenly


def shard_range(n_items: int, rank: int, world: int) -> range:
    """Contiguous shard of [0, n_items) owned by ``rank`` (sizes differ by <= 1)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return split_evenly(n_items, world)[rank]


def shard_blocks(n: int, b_n: int, rank: int, world: int) -> range:
    """Minibatch rows owned by ``rank`` when whole b_n blocks are distributed."""
    if n % b_n:
        raise ValueError(f"b_n={b_n} does not divide N={n}")
    blocks = shard_range(n // b_n, rank, world)
    return range(blocks.start * b_n, blocks.stop * b_n)


@dataclass
class GradientReducer:
    """Per-layer bucketed all-reduce(sum) of gradients on a side stream.

    ``submit(l, tensors)`` enqueues layer ``l``'s gradients as soon as the
    producing pass has been issued; ``wait()`` joins the communication stream
    back into the compute stream before the optimizer step.
    """

    group: object = None
    async_ops: list = field(default_factory=list)
    stream: object = None

    def __post_init__(self):
        import torch

        self._cuda = torch.cuda.is_available()
        if self._cuda and self.stream is None:
            self.stream = torch.cuda.Stream()

    @property
    def world(self) -> int:
        import torch.distributed as dist

        return dist.get_world_size(self.group)

    def submit(self, tensors) -> None:
        import torch
        import torch.distributed as dist

        if self._cuda and tensors and tensors[0].is_cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            self.stream.wait_event(ev)
            with torch.cuda.stream(self.stream):
                for t in tensors:
                    self.async_ops.append(dist.all_reduce(t, group=self.group, async_op=True))
        else:
            for t in tensors:
                self.async_ops.append(dist.all_reduce(t, group=self.group, async_op=True))

    def wait(self) -> None:
        import torch

        for op in self.async_ops:
            op.wait()
        self.async_ops.clear()
        if self._cuda and self.stream is not None:
            torch.cuda.current_stream().wait_stream(self.stream)


def broadcast_params(tensors, group=None) -> None:
    """Make every rank's parameters equal to the group's first rank's (in place)."""
    import torch.distributed as dist

    src = dist.get_global_rank(group, 0) if group is not None and group != dist.group.WORLD else 0
    for t in tensors:
        dist.broadcast(t, src=src, group=group)


def sgd_scale(lr: float, world: int) -> float:
    """Step size applied to the all-reduced SUM so the update uses the global-mean gradient."""
    if world < 1:
        raise ValueError("world must be >= 1")
    return lr / world
