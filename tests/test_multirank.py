"""N>1 host path on the CPU: shard ranges and the result gather, over gloo
with world_size 2 (the GPU box has one GPU; NCCL replaces gloo there)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1001_5272_b200.shard import gather_to_root, local_shard, shard_ranges


def test_shard_ranges_cover_and_balance():
    rng = np.random.default_rng(1)
    lens = rng.integers(2 ** 15 + 1, 2 ** 16 + 1, 4096)
    for world in (1, 2, 3, 4, 8):
        rs = shard_ranges(lens, world)
        assert rs[0][0] == 0 and rs[-1][1] == lens.size
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        sums = [int(lens[s:e].sum()) for s, e in rs]
        assert max(sums) - min(sums) <= 2 * lens.max()
    assert shard_ranges([5], 4)[0] in ((0, 1), (0, 0))
    assert sum(e - s for s, e in shard_ranges([5], 4)) == 1
    assert shard_ranges([], 2) == [(0, 0), (0, 0)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, lens, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, e, ln, off = local_shard(lens, rank, world)
    # each rank "transforms" its shard (here: tags words with the rank) ...
    local = torch.full((int(ln.sum()),), rank + 1, dtype=torch.int32)
    out = gather_to_root(local)
    if rank == 0:
        q.put((out.tolist(), [shard_ranges(lens, world)]))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_two_ranks_gloo():
    lens = [3, 5, 2, 7, 1]
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, lens, q)) for r in range(world)]
    for p in procs:
        p.start()
    out, (ranges,) = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = []
    for r, (s, e) in enumerate(ranges):
        want += [r + 1] * int(sum(lens[s:e]))
    assert out == want


def _worker_transform(rank, world, port, q):
    """Each rank transforms its shard of one ragged batch (the CPU oracle
    stands in for the rank's GPU), then the results are gathered to rank 0
    -- the bench's sharded config-2 path at reduced size."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, top, K = 998244353, pow(3, 119, 998244353), 23
    rng = np.random.default_rng(1)
    lens = rng.integers(1, 3000, 37).astype(np.int64)
    flat = rng.integers(0, p, int(lens.sum()), dtype=np.uint64)
    s, e, ln, off = local_shard(lens, rank, world)
    base = int(np.concatenate(([0], np.cumsum(lens)))[s])
    mine = flat[base:base + int(ln.sum())]
    out = O.tft_batch(mine, ln, p, top, K)
    local = torch.from_numpy(out.astype(np.int64))
    full = gather_to_root(local)
    if rank == 0:
        want = O.tft_batch(flat, lens, p, top, K).astype(np.int64)
        q.put(bool(np.array_equal(full.numpy(), want)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_transform_and_gather_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_transform, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok = q.get(timeout=180)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
