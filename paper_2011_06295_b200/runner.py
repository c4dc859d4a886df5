"""Batch-sharded multi-GPU runner (north-star item 4).

The reference is single-process: its only parallelism is the numba prange
over (image block, output channel) work units whose outputs are disjoint
(_kernels.py:61-72).  Images are independent, so the B200 runner splits the
batch into contiguous per-rank shards -- one process per GPU, weights
replicated (each rank uploads the same CsrKernels) -- and runs the whole
conv stack locally.  There is no collective on the data path; the only one
is the optional final gather of the outputs to rank 0
(``torch.distributed.gather``; NCCL over NVLink on the GPU box, gloo in the
CPU tests).
"""
from __future__ import annotations


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) of rank's contiguous shard of n images; the first
    n % world ranks get one extra image (every image exactly once)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    if n < 0:
        raise ValueError("negative batch")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_sizes(n: int, world: int) -> list[int]:
    return [b - a for a, b in (shard_range(n, world, r) for r in range(world))]


class BatchShardedRunner:
    """Run ``forward(x_shard) -> y_shard`` on this rank's slice of a global
    batch and (optionally) gather every rank's output to rank 0.

    ``forward`` is typically ``SparseConvNet.forward_device`` of a net planned
    for ``shard_sizes(n, world)[rank]`` images.  The process group must be
    initialised (``nccl`` on GPUs; ``gloo`` works for CPU tensors)."""

    def __init__(self, forward, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.forward = forward
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def local_slice(self, n: int) -> slice:
        a, b = shard_range(n, self.world, self.rank)
        return slice(a, b)

    def run(self, x_global_or_shard, n: int | None = None, gather: bool = True):
        """If `n` is given, `x_global_or_shard` is the global batch (every rank
        holds it, e.g. the same host array) and this rank slices its shard;
        otherwise it is already this rank's shard.  Returns the concatenated
        global output on rank 0 when `gather`, else this rank's output."""
        import torch
        x = x_global_or_shard[self.local_slice(n)] if n is not None else x_global_or_shard
        y = self.forward(x)
        if not gather or self.world == 1:
            return y
        sizes = shard_sizes(n, self.world) if n is not None else self._all_sizes(y)
        if y.is_cuda and self.dist.get_backend(self.group) == "gloo":
            y = y.cpu()  # gloo gathers host tensors (CPU tests, oversubscribed single-GPU runs)
        # gather needs equal shapes: pad every shard to the largest
        m = max(sizes)
        yp = y
        if y.shape[0] < m:
            yp = torch.cat([y, y.new_zeros((m - y.shape[0], *y.shape[1:]))])
        bufs = [torch.empty_like(yp) for _ in range(self.world)] if self.rank == 0 else None
        self.dist.gather(yp.contiguous(), bufs, dst=0, group=self.group)
        if self.rank != 0:
            return None
        return torch.cat([b[:s] for b, s in zip(bufs, sizes)])

    def _all_sizes(self, y):
        import torch
        dev = "cpu" if self.dist.get_backend(self.group) == "gloo" else y.device
        t = torch.tensor([y.shape[0]], dtype=torch.int64, device=dev)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [int(v.item()) for v in out]
