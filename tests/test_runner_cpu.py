"""Batch-sharded runner logic on CPU: shard arithmetic and a world_size-2
gloo run whose gathered output equals the single-process result."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_06295_b200.runner import BatchShardedRunner, shard_range, shard_sizes


@pytest.mark.parametrize("n,world", [(256, 1), (256, 2), (256, 8), (7, 3), (3, 8), (0, 4)])
def test_shards_cover_batch_once(n, world):
    seen = []
    for r in range(world):
        a, b = shard_range(n, world, r)
        assert 0 <= a <= b <= n
        seen.extend(range(a, b))
    assert seen == list(range(n))
    sizes = shard_sizes(n, world)
    assert max(sizes) - min(sizes) <= 1


def test_bad_rank():
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _forward(x):
    # stand-in for SparseConvNet.forward_device: per-image, batch-independent
    return torch.relu(x * 2.0 - 1.0).sum(dim=(2, 3))


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(0)
        x = torch.randn((n, 3, 4, 4), generator=g)  # every rank holds the same global batch
        out = BatchShardedRunner(_forward).run(x, n=n)
        if rank == 0:
            q.put(out.numpy())
        # shards passed directly (sizes exchanged by all_gather)
        sl = slice(*shard_range(n, world, rank))
        out2 = BatchShardedRunner(_forward).run(x[sl])
        if rank == 0:
            q.put(out2.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [8, 7])
def test_gloo_world2_gather_matches_single_process(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    a = q.get(timeout=120)
    b = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = torch.Generator().manual_seed(0)
    ref = _forward(torch.randn((n, 3, 4, 4), generator=g)).numpy()
    assert (a == ref).all() and (b == ref).all()
