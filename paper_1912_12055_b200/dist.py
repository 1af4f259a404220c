"""Multi-GPU plumbing: one process per GPU.

The forward path shards clips across ranks with no collective (outputs stay
sharded).  Trainable layers need exactly one exchange per step: the sum of
the kernel / mel-weight gradients over ranks (NCCL all-reduce over NVLink on
B200; gloo in the CPU tests).  `GradReducer` buckets it by readiness inside
the backward pass -- the mel-weight gradient as soon as its GEMM finishes
(overlapping the coef and dK GEMMs), the first 1,024 DFT-bank rows while the
rest of dK runs, the remainder last -- and `allreduce_grads` is the one-bucket
form.  The summation order is fixed by NCCL's ring/tree for a given world
size, so runs are reproducible.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_rank_world() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of n_items for `rank`: the first n % world
    ranks get one extra item (1770 clips on 8 GPUs -> 222, 222, 221 x 6)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_batch(x: torch.Tensor, rank: int | None = None, world: int | None = None) -> torch.Tensor:
    """This rank's clips of a (B, L) batch."""
    if rank is None or world is None:
        rank, world, _ = env_rank_world()
    lo, hi = shard_range(int(x.shape[0]), rank, world)
    return x[lo:hi]


def allreduce_grads(params, group=None, average: bool = False) -> None:
    """Sum (or average) .grad of `params` over the process group with ONE
    flattened all-reduce (a single bucket: the per-step traffic of the
    trainable STFT+Mel layer is 17.3 MB)."""
    if not dist.is_available() or not dist.is_initialized():
        return
    grads = [p.grad for p in params if p.grad is not None]
    if not grads:
        return
    flat = torch.cat([g.reshape(-1) for g in grads])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    if average:
        flat /= dist.get_world_size(group)
    off = 0
    for g in grads:
        n = g.numel()
        g.copy_(flat[off:off + n].view_as(g))
        off += n


def gather_shards(y: torch.Tensor, n_items: int, group=None) -> torch.Tensor:
    """Reassemble a clip-sharded output (only for checks; the bench keeps outputs sharded)."""
    world = dist.get_world_size(group)
    sizes = [shard_range(n_items, r, world) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((width,) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
    pad[: y.shape[0]] = y
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, sizes)])


class GradReducer:
    """Bucketed all-reduce (sum) of the gradients a trainable layer's backward
    produces, each bucket launched asynchronously the moment its GEMM has been
    issued (NCCL's stream waits for the compute stream at launch, so the
    reduction of bucket i overlaps the GEMMs that produce bucket i+1).

    Protocol with `autograd.DftLayerOp.backward`: while armed, the op calls
    `launch(t)` for every finished gradient block and `wait()` before it
    returns, so the compute stream is ordered after every reduction before
    autograd accumulates the gradients (no stream race on .grad)."""

    def __init__(self, module_or_ops, group=None):
        from .autograd import DftLayerOp
        if isinstance(module_or_ops, torch.nn.Module):
            ops = []
            for m in module_or_ops.modules():
                op = getattr(m, "_op", None)
                if isinstance(op, DftLayerOp) and op not in ops:
                    ops.append(op)
        else:
            ops = list(module_or_ops)
        self.ops, self.group, self.works, self.buckets = ops, group, [], 0

    def arm(self):
        for op in self.ops:
            op.reducer = self
        self.works, self.buckets = [], 0

    def launch(self, t: torch.Tensor):
        if dist.is_available() and dist.is_initialized():
            self.works.append(dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        self.buckets += 1

    def wait(self):
        for w in self.works:
            w.wait()
        self.works = []

    def finish(self):
        self.wait()
        for op in self.ops:
            op.reducer = None
