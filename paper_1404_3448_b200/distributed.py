"""Multi-GPU plumbing for batched pairs (BASELINE config C4).

Independent pairs shard contiguously across ranks (one process per GPU);
every rank runs its shard through ``OverlapBatch`` and the per-pair results
(3 x int64 per pair) are all-gathered -- the only collective of the path: on
GPUs by NCCL inside libsaix_b200.so (``NcclComm``, saix_comm_* in the C ABI),
torch.distributed only bootstrapping the NCCL id; the CPU tests run the same
gather over a gloo process group (``gather_results``).
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
    # gloo gathers host tensors (CPU tests, or several ranks sharing one GPU)
    host = local.is_cuda and dist.get_backend(group) == "gloo"
    src = local.cpu() if host else local
    mine = src.new_zeros(width)
    mine[: src.numel()].copy_(src.reshape(-1))
    parts = [src.new_empty(width) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    full = torch.cat([p[: 3 * c] for p, c in zip(parts, counts)]).reshape(total, 3)
    return full.to(local.device) if host else full


class NcclComm:
    """This rank's NCCL communicator held by libsaix_b200.so (saix_comm_*):
    the result all-gather and the first-error MIN all-reduce run inside the
    library on the current stream, PyTorch supplies device buffers only.
    ``dist`` (any torch.distributed backend) is used once, to broadcast rank
    0's 128-byte NCCL id (the bootstrap)."""

    def __init__(self, dist, world: int, rank: int, device: int | None = None, group=None):
        import ctypes

        import torch

        from . import _lib
        L = _lib.load()
        self.world, self.rank = world, rank
        dev = torch.cuda.current_device() if device is None else device
        idb = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _lib.check(L.saix_comm_unique_id(idb), "saix_comm_unique_id")
        box = [bytes(idb)]
        if dist is not None and world > 1:
            dist.broadcast_object_list(box, src=0, group=group)
        idb = (ctypes.c_uint8 * 128).from_buffer_copy(box[0])
        self._comm = ctypes.c_void_p()
        _lib.check(L.saix_comm_init(ctypes.byref(self._comm), world, idb, rank, dev), "saix_comm_init")

    def all_gather(self, send):
        """(world * send.numel()) int64 device tensor: every rank's block in rank order."""
        import torch

        from . import _lib
        out = torch.empty(self.world * send.numel(), dtype=torch.int64, device=send.device)
        _lib.check(_lib.load().saix_comm_allgather_i64(self._comm, _lib.ptr(send), send.numel(), _lib.ptr(out),
                                                       _lib.stream_ptr()), "saix_comm_allgather_i64")
        return out

    def all_reduce_min(self, t):
        from . import _lib
        out = t.clone()
        _lib.check(_lib.load().saix_comm_allreduce_min_i64(self._comm, _lib.ptr(t), _lib.ptr(out), t.numel(),
                                                           _lib.stream_ptr()), "saix_comm_allreduce_min_i64")
        return out

    def close(self):
        from . import _lib
        if self._comm:
            _lib.check(_lib.load().saix_comm_destroy(self._comm), "saix_comm_destroy")
            self._comm = None

    def __del__(self):
        import sys
        if sys.is_finalizing():  # the CUDA runtime may already be gone: let the process exit free it
            return
        try:
            self.close()
        except Exception:
            pass


def gather_results_nccl(local, total: int, world: int, comm: NcclComm):
    """gather_results over the library's NCCL communicator (device tensors)."""
    import torch
    counts = [hi - lo for lo, hi in (shard(total, world, r) for r in range(world))]
    width = 3 * max(counts)
    mine = torch.zeros(width, dtype=torch.int64, device=local.device)
    mine[: local.numel()].copy_(local.reshape(-1))
    allr = comm.all_gather(mine).view(world, width)
    return torch.cat([allr[r, : 3 * c] for r, c in enumerate(counts)]).reshape(total, 3)


class ShardedOverlapBatch:
    """This rank's shard of a batched longest-overlap job plus the gather.

    `policy` is the reference's NPolicy (REJECT by default, as in
    `longest_overlap`, overlap.py:110): an illegal residue anywhere in the job
    raises the reference's SequenceError on every rank -- the ranks agree on
    the smallest offending pair (all-reduce MIN) before any result is
    gathered, so no rank returns overlaps computed past a bad residue."""

    def __init__(self, seqs, offs, total: int, world: int, rank: int, dist=None, group=None,
                 policy=None, comm: NcclComm | None = None):
        from .overlap import OverlapBatch
        from .sequence import NPolicy
        self.total, self.world, self.rank = total, world, rank
        self.dist, self.group, self.comm = dist, group, comm
        self.lo, self.hi = shard(total, world, rank)
        self.policy = NPolicy.REJECT if policy is None else policy
        self.batch = OverlapBatch(seqs, offs, self.policy)
        if self.batch.P != self.hi - self.lo:
            raise ValueError("seqs/offs must hold exactly this rank's shard")

    def _first_bad(self):
        """(global sequence index 2p+side, offset in that sequence) of the
        first illegal residue over all ranks, or None."""
        import numpy as np
        import torch
        from .overlap import INT64_MAX
        b = self.batch
        key = INT64_MAX
        pos = b.first_bad()                                           # offset in this rank's seqs
        if pos is not None:
            si = int(np.searchsorted(b.offs, pos, side="right") - 1)  # sequence 2p or 2p+1 of the shard
            key = ((2 * self.lo + si) << 40) | (pos - int(b.offs[si]))
        if self.comm is not None and self.world > 1:
            key = int(self.comm.all_reduce_min(torch.tensor([key], dtype=torch.int64, device=b.bad.device)).item())
        elif self.dist is not None and self.world > 1:
            on = "cpu" if self.dist.get_backend(self.group) == "gloo" else b.bad.device
            t = torch.tensor([key], dtype=torch.int64, device=on)
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
            key = int(t.item())
        return None if key == INT64_MAX else (key >> 40, key & ((1 << 40) - 1))

    def check(self, seq_of=None):
        """Raise the reference's SequenceError for the first illegal residue
        of the whole job, identically on every rank.  `seq_of(g)` returns
        DnaSequence g (= 2 * pair + side) for encode()'s exact message;
        without it the message names the pair, side and offset."""
        from .sequence import SequenceError, residue_error
        hit = self._first_bad()
        if hit is None:
            return
        g, off = hit
        if seq_of is not None:
            raise residue_error(seq_of(g), off, self.policy)
        raise SequenceError(f"pair {g // 2} sequence {'AB'[g % 2]}: illegal residue at position {off} "
                            f"(policy={self.policy.value})")

    def run(self, seq_of=None):
        """Run the shard; returns the (total, 3) result tensor (device).
        Raises SequenceError (on every rank) if any rank saw an illegal
        residue under REJECT."""
        self.batch.run_device()
        self.check(seq_of)
        local = self.batch.out[: 3 * self.batch.P]
        if self.world == 1:
            return local.reshape(-1, 3)
        if self.comm is not None:
            return gather_results_nccl(local, self.total, self.world, self.comm)
        return gather_results(local, self.total, self.world, self.dist, self.group)
