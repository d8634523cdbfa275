"""Batch sharding across GPUs (one process per GPU, torch.distributed).

The path partitions: vectors (and products) are independent, so a batch is
split into contiguous ranges balanced by total words, each rank transforms
its range with no data-path collective, and an optional gather brings
results to one rank afterwards (outside the transform; the reference has no
collective at all).
"""

import numpy as np


def shard_ranges(lengths, world):
    """Contiguous [start, end) vector ranges, one per rank, balanced by the
    sum of lengths (greedy prefix cut at multiples of total/world).  Every
    vector lands in exactly one range; ranges may be empty when there are
    fewer vectors than ranks."""
    ln = np.asarray(lengths, dtype=np.int64)
    if world < 1:
        raise ValueError("world must be >= 1")
    if ln.size == 0:
        return [(0, 0)] * world
    csum = np.cumsum(ln)
    total = int(csum[-1])
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        i = int(np.searchsorted(csum, target, side="left"))  # csum[i] >= target
        lo = int(csum[i - 1]) if i > 0 else 0                # words before a cut after i vectors
        hi = int(csum[i]) if i < ln.size else total          # ... after i+1 vectors
        c = i if target - lo <= hi - target else i + 1
        cuts.append(max(cuts[-1], min(c, ln.size)))
    cuts.append(ln.size)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def local_shard(lengths, rank, world):
    """(start, end, local lengths, local offsets relative to the shard)."""
    s, e = shard_ranges(lengths, world)[rank]
    ln = np.asarray(lengths, dtype=np.int64)[s:e]
    off = np.concatenate(([0], np.cumsum(ln)[:-1])).astype(np.int64) if ln.size else ln
    return s, e, ln, off


def gather_to_root(local, group=None, root=0):
    """Gather variable-length 1-D tensors from every rank onto `root` (pads to
    the longest shard; works with gloo on CPU and NCCL on CUDA).  Returns the
    concatenation on root, None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = torch.tensor([local.numel()], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    m = int(max(s.item() for s in sizes))
    buf = torch.zeros(m, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    if dist.get_rank(group) == root:
        parts = [torch.zeros(m, dtype=local.dtype, device=local.device) for _ in range(world)]
        dist.gather(buf, parts, dst=root, group=group)
        return torch.cat([p[: int(s.item())] for p, s in zip(parts, sizes)])
    dist.gather(buf, None, dst=root, group=group)
    return None
