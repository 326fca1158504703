"""Multi-GPU plumbing for batched pairs (BASELINE config C4).

Independent pairs shard contiguously across ranks (one process per GPU);
every rank runs its shard through ``OverlapBatch`` and the per-pair results
(3 x int64 per pair) are all-gathered -- the only collective of the path (NCCL
over NVLink on GPUs; any torch.distributed backend works, the tests use gloo).
"""

from __future__ import annotations


def shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of `total` pairs for `rank` (pairs
    [g P/G, (g+1) P/G) on rank g)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return total * rank // world, total * (rank + 1) // world


def gather_results(local, total: int, world: int, dist, group=None):
    """All-gather every rank's (P_r * 3) int64 result tensor into the full
    (total, 3) tensor in pair order, on every rank.  Shards differ by at most
    one pair, so each rank pads to the largest shard for the collective."""
    import torch
    counts = [hi - lo for lo, hi in (shard(total, world, r) for r in range(world))]
    width = 3 * max(counts)
    mine = local.new_zeros(width)
    mine[: local.numel()].copy_(local.reshape(-1))
    parts = [local.new_empty(width) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    return torch.cat([p[: 3 * c] for p, c in zip(parts, counts)]).reshape(total, 3)


class ShardedOverlapBatch:
    """This rank's shard of a batched longest-overlap job plus the gather."""

    def __init__(self, seqs, offs, total: int, world: int, rank: int, dist=None, group=None):
        from .overlap import OverlapBatch
        self.total, self.world, self.rank = total, world, rank
        self.dist, self.group = dist, group
        self.lo, self.hi = shard(total, world, rank)
        self.batch = OverlapBatch(seqs, offs)
        if self.batch.P != self.hi - self.lo:
            raise ValueError("seqs/offs must hold exactly this rank's shard")

    def run(self):
        """Run the shard; returns the (total, 3) result tensor (device)."""
        self.batch.run_device()
        local = self.batch.out[: 3 * self.batch.P]
        if self.dist is None or self.world == 1:
            return local.reshape(-1, 3)
        return gather_results(local, self.total, self.world, self.dist, self.group)
