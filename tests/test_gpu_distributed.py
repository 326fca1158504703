"""Two ranks on one B200 (gloo for the host plumbing; NCCL refuses two ranks
on one device): ShardedOverlapBatch end to end -- contiguous shards of C4
pairs, per-pair results gathered in pair order on every rank -- against the
C oracle, and the REJECT policy raising the same SequenceError on every rank
when only one rank's shard holds an illegal residue (reference
overlap.py:110-152 per pair, sequence.py:152-156 for the error)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, poison, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1404_3448_b200.distributed import ShardedOverlapBatch, shard
        from paper_1404_3448_b200.sequence import SequenceError
        from paper_1404_3448_b200.workloads import c4_pairs
        lo, hi = shard(total, world, rank)
        seqs, offs = c4_pairs(lo, hi)
        if poison is not None and lo <= poison[0] < hi:
            p, side, off = poison
            seqs = seqs.copy()
            seqs[offs[2 * (p - lo) + side] + off] = ord("X")
        job = ShardedOverlapBatch(seqs, offs, total, world, rank, dist)
        try:
            full = job.run()
            q.put((rank, "ok", full.cpu().numpy().tolist()))
        except SequenceError as e:
            q.put((rank, "err", str(e)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(world, total, poison=None):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, poison, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


def test_sharded_batch_two_ranks_matches_oracle():
    import oracle
    from paper_1404_3448_b200.workloads import c4_pairs
    total = 601
    out = _run(2, total)
    seqs, offs = c4_pairs(0, total)
    want = oracle.overlap_batch(seqs, offs, threads=os.cpu_count() or 1).tolist()
    for rank, kind, full in out:
        assert kind == "ok"
        assert full == want


def test_sharded_batch_reject_raises_on_every_rank():
    total = 40
    out = _run(2, total, poison=(33, 1, 17))   # pair 33 lives on rank 1
    msgs = {m for _, kind, m in out if kind == "err"}
    assert len(msgs) == 1 and all(kind == "err" for _, kind, _ in out)
    assert "pair 33 sequence B" in msgs.pop()


def test_library_nccl_comm_single_rank():
    """The C-ABI collective (saix_comm_*: NCCL bound inside libsaix_b200.so)
    on one device: id, init, all-gather, MIN all-reduce, and a world-1
    ShardedOverlapBatch gather through it against the oracle."""
    import torch

    import oracle
    from paper_1404_3448_b200.distributed import NcclComm, ShardedOverlapBatch, gather_results_nccl
    from paper_1404_3448_b200.workloads import c4_pairs
    torch.cuda.set_device(0)
    comm = NcclComm(None, 1, 0)
    x = torch.arange(12, dtype=torch.int64, device="cuda")
    assert torch.equal(comm.all_gather(x), x)
    assert torch.equal(comm.all_reduce_min(x), x)
    assert torch.equal(gather_results_nccl(x, 4, 1, comm), x.reshape(4, 3))
    seqs, offs = c4_pairs(0, 30)
    job = ShardedOverlapBatch(seqs, offs, 30, 1, 0, comm=comm)
    got = job.run().cpu().numpy()
    assert np.array_equal(got, oracle.overlap_batch(seqs, offs))
    comm.close()
