"""Batch-sharded data parallelism for the PSN layer.

One process per GPU (``torchrun``), ``torch.distributed`` for the plumbing.
Every element's convolution is independent across the batch axis
(reference engines.py:132 acts per (n, c)), so each rank runs the neuron
layer on its contiguous batch shard with no data-path collective.  The
only exchange is the per-channel parameter gradients (dW [C,k], dgamma
[C], dbeta [C] -- 12 KB at C=512, k=4), all-reduced in one flat bucket
after the backward.

Semantics: batch statistics are per shard (standard DDP without SyncBN),
so a rank's spikes and dx equal the reference run on that shard, and the
summed gradients equal the sum of the per-shard reference gradients.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) of the batch rows rank `rank` owns; the first
    `batch % world` ranks take one extra row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"invalid rank {rank} of world {world}")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_batch(x: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """This rank's slice of a time-first tensor [T, N, C, ...] along N."""
    a, b = shard_bounds(x.shape[1], rank, world)
    return x[:, a:b]


class GradBucket:
    """One flat buffer over a fixed list of parameters: gradients are packed,
    all-reduced with a single collective and unpacked (bucketed DDP)."""

    def __init__(self, params):
        self.params = [p for p in params if p.requires_grad]
        if not self.params:
            raise ValueError("no parameters to reduce")
        dev = self.params[0].device
        dtypes = {p.dtype for p in self.params}
        if len(dtypes) != 1:
            raise ValueError(f"parameters of one bucket share a dtype, got {dtypes}")
        self.numels = [p.numel() for p in self.params]
        self.flat = torch.zeros(sum(self.numels), dtype=self.params[0].dtype, device=dev)

    def views(self) -> list:
        """Per-parameter views into the flat buffer, shaped like the parameters:
        a backward that writes its gradients straight into them needs no pack
        step before `reduce_()` (zero-copy bucket, as bench.py's step does)."""
        out, off = [], 0
        for p, n in zip(self.params, self.numels):
            out.append(self.flat[off:off + n].view_as(p))
            off += n
        return out

    def reduce_(self, group=None, average: bool = False) -> torch.Tensor:
        """All-reduce the flat buffer in place (no pack / unpack)."""
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)
            if average:
                self.flat.div_(dist.get_world_size(group))
        return self.flat

    def pack(self) -> torch.Tensor:
        off = 0
        for p, n in zip(self.params, self.numels):
            g = p.grad
            self.flat[off:off + n].copy_(g.reshape(-1) if g is not None else torch.zeros(n, dtype=p.dtype))
            off += n
        return self.flat

    def unpack(self) -> None:
        off = 0
        for p, n in zip(self.params, self.numels):
            view = self.flat[off:off + n].view_as(p)
            if p.grad is None:
                p.grad = view.clone()
            else:
                p.grad.copy_(view)
            off += n

    def allreduce(self, group=None, average: bool = False) -> None:
        """Sum (or average) the bucket across the process group in place."""
        self.pack()
        self.reduce_(group=group, average=average)
        self.unpack()


def allreduce_grads(params, group=None, average: bool = False) -> None:
    """Convenience wrapper: one bucket, one all-reduce."""
    GradBucket(params).allreduce(group=group, average=average)
