#!/usr/bin/env python
"""Benchmark of the B200 longest-overlap hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c3|c5]

Default workload (BASELINE.json configs[1], "C2"): one synthetic pair of
2 x 10 Mbp random ACGT sequences (gen_random seeds 11/12 on rank 0; rank r
uses 11+2r/12+2r), full pipeline on one B200 per rank: encode -> generalized
text -> DC3 suffix array -> LCP -> overlap scan.  A "step" is one pass of the
pipeline over one pair.  Metric: Mbases/s of generalized-text bases through
the whole pipeline (20,000,001 per pair); `value` is the whole-job aggregate;
N > 1 runs independent replicas (weak scaling, no data-path collective: a
single long pair does not shard).

Other BASELINE configs (reported in DESIGN.md / profiles/, not the default):
  c3  configs[2]: 256 Mbp (2^28) DC3 suffix array + LCP, Mbases/s
  c5  configs[4]: 10^8 random sparse-table RMQ queries over the LCP array of a
      64 Mbp (2^26) text, table build + queries per step, queries/s

--impl reference times the reference algorithm on the host (the C oracle port
in oracle/, kind "port": the reference is pure Python + numba, nothing to
compile) on the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DC3 suffix-array Mbases/s; longest-overlap pairs/s at 1/2/4/8 B200 vs host CPU"
L2_FLUSH_BYTES = 512 << 20


# ------------------------------------------------------------------ helpers

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peak_gbs():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML
    polled every 2 ms from a thread (nvidia-smi -lms as the fallback)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[float, float, int]] = []
        self.stop_flag = threading.Event()
        self.nvml = None
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            try:  # the CUDA device's PCI address (CUDA_VISIBLE_DEVICES may renumber)
                import torch
                pr = torch.cuda.get_device_properties(self.index)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (pynvml, h)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _poll(self):
        pynvml, h = self.nvml
        smax = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        while not self.stop_flag.is_set():
            try:
                sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                try:
                    rs = int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
                except Exception:
                    rs = int(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h))
                self.samples.append((sm, smax, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.t.join(timeout=2)
            sm = [x[0] for x in self.samples]
            reasons = sorted({nm for _, _, rs in self.samples for nm, bit in self.REASONS.items() if rs & bit})
            return {"sm_mhz": statistics.median(sm) if sm else None,
                    "sm_max_mhz": self.samples[0][1] if self.samples else None,
                    "reasons": reasons, "samples": len(sm), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


def count_our_launches(fn) -> int:
    """Kernels from libsaix_b200 (all named k_*) launched by one call of fn."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    n = 0
    for e in prof.events():
        name = e.name or ""
        if e.device_type.name == "CUDA" and ("k_" in name.split("(")[0].split("<")[0]):
            n += 1
    return n


def ncu_traffic(workload: str, scope: str):
    """DRAM read+write bytes per invocation of the prof scope `scope` from the
    committed ncu launch-list summary (profiles/ncu_traffic.json, written by
    tools/make_traffic.py from `ncu --metrics dram__bytes_read.sum,
    dram__bytes_write.sum,...` of one step of the same workload), if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload, {}).get(scope)
    except Exception:
        return None


def dc3_model_bytes(trace, isa: bool = False) -> float:
    """SURVEY.md section 8(d) contract: algorithmic DC3 bytes over the level
    trace (N, sigma, m, names) -- per level (k = ceil(N/3), r = recurses,
    w = 1 at level 0 and 4 below): (wN + 8m) + 72m + 16m + 8m r + (4m + (12+w)k)
    + (4m + 4k + (2w+8)N), plus 8n for a top-level ISA."""
    total = 0.0
    for lvl, (n_l, _sigma, m, names) in enumerate(trace):
        w = 1 if lvl == 0 else 4
        k = (n_l + 2) // 3
        r = 1 if names < m else 0
        total += (w * n_l + 8 * m) + 72 * m + 16 * m + 8 * m * r + (4 * m + (12 + w) * k) \
            + (4 * m + 4 * k + (2 * w + 8) * n_l)
    if isa and trace:
        total += 8 * trace[0][0]
    return total


def encode_ascii(residues: str, shift: int = 0) -> np.ndarray:
    lut = np.zeros(256, np.uint8)
    for r, ch in enumerate("ACGT", 1 + shift):
        lut[ord(ch)] = r
    return lut[np.frombuffer(residues.encode(), np.uint8)]


# ------------------------------------------------------------------ workloads

class C2:
    """configs[1]: full longest-overlap pipeline on one 2 x 10 Mbp pair."""
    name = "c2"
    unit = "Mbases/s"

    def __init__(self, rank: int):
        from paper_1404_3448_b200.sequence import gen_random
        import paper_1404_3448_b200 as sx
        a = gen_random(10_000_000, 11 + 2 * rank)
        b = gen_random(10_000_000, 12 + 2 * rank)
        self.ha = np.frombuffer(a.residues.encode(), np.uint8)
        self.hb = np.frombuffer(b.residues.encode(), np.uint8)
        self.units = len(self.ha) + len(self.hb) + 1          # GSA bases per step
        self.pipe = sx.OverlapPipeline(len(self.ha), len(self.hb))
        self.pipe.stage(self.ha, self.hb)
        self.result = [int(x) for x in self.pipe.run_staged()[:3]]
        self.h2d = len(self.ha) + len(self.hb)
        self.d2h = 32
        self.config = {"workload": "C2: 2 x 10 Mbp random ACGT pair (gen_random seeds 11/12 + 2*rank), "
                                   "encode+DC3+LCP+overlap scan per step",
                       "gsa_bases_per_pair": self.units}

    def step_device(self):
        self.pipe.run_device()

    def step_e2e(self):
        self.pipe.run_staged()

    def extra(self, ms_dev, steps, world):
        return {"pairs_per_s": round(world * steps / (ms_dev * 1e-3), 3)}

    def cpu_baseline(self):
        import oracle
        t0 = time.perf_counter()
        ref = oracle.longest_overlap(self.ha.tobytes(), self.hb.tobytes())
        dt = time.perf_counter() - t0
        assert tuple(self.result) == ref, (self.result, ref)
        return {"value": self.units / dt / 1e6, "unit": self.unit, "cores": 1, "kind": "port",
                "sample": "one full C2 pair (2 x 10 Mbp), oracle/saix_oracle.c single thread "
                          f"({dt:.1f} s); result matched the GPU's {tuple(ref)}"}


class C3:
    """configs[2]: DC3 suffix array + LCP of a 2^28 random text."""
    name = "c3"
    unit = "Mbases/s"
    N = 1 << 28

    def __init__(self, rank: int):
        from paper_1404_3448_b200.sequence import gen_random
        from paper_1404_3448_b200.suffix_index import SuffixIndexer
        self.ranks = encode_ascii(gen_random(self.N, 1 + rank).residues)
        self.units = self.N
        self.ix = SuffixIndexer(self.N, 4)
        self.ix.stage(self.ranks)
        self.ix.run_staged()
        self.h2d = self.N
        self.d2h = 8 * self.N
        self.config = {"workload": "C3: 2^28 random ACGT (gen_random seed 1 + rank), DC3 suffix array + LCP "
                                   "per step (SA and LCP u32 resident; e2e downloads both)",
                       "bases": self.N}
        self.result = None

    def step_device(self):
        self.ix.run_device()

    def step_e2e(self):
        self.ix.run_staged()

    def extra(self, ms_dev, steps, world):
        return {}

    def cpu_baseline(self):
        import oracle
        # bounded sample: DC3 + Kasai of the first 2^24 bases (~10-20 s)
        n = 1 << 24
        t = self.ranks[:n].astype(np.int64)
        t0 = time.perf_counter()
        sa, rank = oracle.dc3(t, 4)
        oracle.lcp(t, sa, rank)
        dt = time.perf_counter() - t0
        return {"value": n / dt / 1e6, "unit": self.unit, "cores": 1, "kind": "port",
                "sample": f"DC3 + LCP of the first 2^24 bases of the C3 text, single thread ({dt:.1f} s)"}


class C5:
    """configs[4]: 10^8 random LCP range-minimum queries over a 2^26 text."""
    name = "c5"
    unit = "queries/s"
    N = 1 << 26
    Q = 100_000_000

    def __init__(self, rank: int):
        import torch

        from paper_1404_3448_b200.rmq import DeviceSparseTable
        from paper_1404_3448_b200.sequence import gen_random
        from paper_1404_3448_b200.suffix_index import SuffixIndexer
        self.ranks = encode_ascii(gen_random(self.N, 1 + rank).residues)
        self.ix = SuffixIndexer(self.N, 4)
        self.ix.stage(self.ranks)
        self.ix.run_staged()
        self.st = DeviceSparseTable(self.ix.lcp, 4, self.N)
        q = np.random.default_rng(2026 + rank).integers(0, self.N, size=(self.Q, 2))
        self.hqi = torch.from_numpy(np.ascontiguousarray(q[:, 0])).pin_memory()
        self.hqj = torch.from_numpy(np.ascontiguousarray(q[:, 1])).pin_memory()
        dev = self.ix.lcp.device
        self.qi = self.hqi.to(dev)
        self.qj = self.hqj.to(dev)
        self.hout = torch.empty(self.Q, dtype=torch.int64, pin_memory=True)
        self.units = self.Q
        self.h2d = 16 * self.Q
        self.d2h = 8 * self.Q
        self.config = {"workload": "C5: sparse-table build over the LCP array of a 2^26 random text + 10^8 "
                                   "query_sparse (default_rng(2026).integers(0, n, (10^8, 2))) per step",
                       "n": self.N, "queries": self.Q, "table_mode": int(self.st.plan.mode)}
        self.out = None
        self.result = None

    def step_device(self):
        self.st.rebuild()
        self.out, _ = self.st.query_device(self.qi, self.qj)

    def step_e2e(self):
        import torch
        self.qi.copy_(self.hqi, non_blocking=True)
        self.qj.copy_(self.hqj, non_blocking=True)
        self.st.rebuild()
        out, _ = self.st.query_device(self.qi, self.qj)
        self.hout.copy_(out, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    def extra(self, ms_dev, steps, world):
        return {}

    def cpu_baseline(self):
        import oracle
        # parity on a 10^6 prefix of the queries against the leftmost-argmin definition
        lcp = self.ix.lcp[: self.N].cpu().numpy().view(np.uint32).astype(np.int64)
        qi, qj = self.hqi[:1_000_000].numpy(), self.hqj[:1_000_000].numpy()
        got = self.out[:1_000_000].cpu().numpy()
        assert np.array_equal(got, oracle.argmin_blocked(lcp, qi, qj))
        # timed: the reference SparseTable.query restated in C, over a bounded
        # sample (table of the first 2^22 LCP values, 10^6 queries inside it)
        m = 1 << 22
        v = lcp[:m]
        table = oracle.sparse_build(v)
        rng = np.random.default_rng(2026)
        si, sj = rng.integers(0, m, size=(2, 1_000_000))
        t0 = time.perf_counter()
        oracle.sparse_query(v, table, si, sj)
        dt = time.perf_counter() - t0
        return {"value": 1_000_000 / dt, "unit": self.unit, "cores": 1, "kind": "port",
                "sample": "10^6 SparseTable.query over the first 2^22 LCP values (C port of rmq.py:52-58), "
                          f"single thread ({dt:.2f} s); GPU answers matched the argmin oracle on 10^6 queries"}


def _c4_chunk(args):
    from paper_1404_3448_b200.workloads import c4_pairs
    return c4_pairs(*args)


class C4:
    """configs[3]: 100k synthetic 10 kbp noncoding-like pairs (workloads.py),
    sharded contiguously across ranks (strong scaling); the per-pair results
    are all-gathered to every rank over NCCL inside the step (the one
    collective of the path)."""
    name = "c4"
    unit = "pairs/s"
    scaling = "strong"
    TOTAL = 100_000

    def __init__(self, rank: int, world: int = 1, dist=None):
        import concurrent.futures as cf

        import torch

        import paper_1404_3448_b200 as sx
        from paper_1404_3448_b200.workloads import shard
        lo, hi = shard(self.TOTAL, world, rank)
        chunks = [(a, min(a + 1000, hi)) for a in range(lo, hi, 1000)]
        with cf.ProcessPoolExecutor(max_workers=min(32, os.cpu_count() or 4)) as ex:
            parts = list(ex.map(_c4_chunk, chunks))
        self.seqs = np.concatenate([p[0] for p in parts])
        offs, base = [np.zeros(1, np.int64)], 0
        for s, o in parts:
            offs.append(o[1:] + base)
            base += int(o[-1])
        self.offs = np.concatenate(offs)
        self.P = hi - lo
        self.dist, self.world = dist, world
        self.ob = sx.OverlapBatch(self.seqs, self.offs)
        self.hseqs = torch.from_numpy(self.seqs).pin_memory()
        self.hout = torch.empty(3 * self.P, dtype=torch.int64, pin_memory=True)
        self.units = self.TOTAL / world
        self.units_total = self.TOTAL
        self.h2d = int(self.seqs.nbytes)
        self.d2h = 24 * self.P
        self.ob.run_device()
        self.result = None
        self.config = {"workload": "C4: 100k pairs of 2 x 10 kbp AT-rich random sequences with one planted "
                                   "shared block (paper_1404_3448_b200/workloads.py), batched waves of <= 2^27 "
                                   "residues, results all-gathered over NCCL",
                       "pairs": self.TOTAL, "pairs_this_rank": self.P, "waves_this_rank": len(self.ob.waves)}
        self.dc3_calls_per_step = len(self.ob.waves)

    def _gather(self):
        if self.dist is None:
            return
        from paper_1404_3448_b200.distributed import gather_results
        self.full = gather_results(self.ob.out[: 3 * self.P], self.TOTAL, self.world, self.dist)

    def step_device(self):
        self.ob.run_device()
        self._gather()

    def step_e2e(self):
        import torch
        self.ob.seqs_dev[: self.seqs.shape[0]].copy_(self.hseqs, non_blocking=True)
        self.ob.run_device()
        self._gather()
        self.hout.copy_(self.ob.out[: 3 * self.P], non_blocking=True)
        torch.cuda.current_stream().synchronize()

    def extra(self, ms_dev, steps, world):
        return {}

    def cpu_baseline(self):
        import oracle
        k = 4000  # bounded sample: the first 4000 pairs on every host thread
        threads = os.cpu_count() or 1
        t0 = time.perf_counter()
        want = oracle.overlap_batch(self.seqs[: self.offs[2 * k]], self.offs[: 2 * k + 1], threads=threads)
        dt = time.perf_counter() - t0
        got = self.ob.results()[:k]
        assert np.array_equal(got, want)
        return {"value": k / dt, "unit": self.unit, "cores": threads, "kind": "port",
                "sample": f"first {k} C4 pairs, oracle/saix_oracle.c on {threads} host threads ({dt:.1f} s); "
                          "GPU answers matched on all of them"}


class Store:
    """.saix save + load round trip (index_store.py:
    65-134) of a 2^26-base index -- device step: fused pack + CRC-32 of the
    file image, then CRC check + decode + ISA rebuild from the image; e2e:
    save_index into a BytesIO and load_index back (host bytes, RMQ rebuild and
    the reference's int64 host arrays included)."""
    name = "store"
    unit = "Mbases/s"
    N = 1 << 26

    def __init__(self, rank: int):
        import torch
        from paper_1404_3448_b200 import _lib, index_store
        from paper_1404_3448_b200.overlap import LcpQueryEngine
        from paper_1404_3448_b200.sequence import encode, gen_random
        from paper_1404_3448_b200.suffix_index import _device_index_of
        n = self.N
        self.ist = index_store
        self.eng = LcpQueryEngine.build(encode(gen_random(n, 21 + rank)))
        self.L = L = _lib.load()
        self.ix = _device_index_of(self.eng.text, self.eng.sa)
        self.lcp = self.eng.lcp._dev[1]
        total = int(L.saix_index_bytes(n))
        self.blob = _lib.empty(total, torch.uint8)
        self.text_d = _lib.empty(n, torch.uint8)
        self.sa_d, self.lcp_d, self.isa_d = (_lib.empty(n, torch.int32) for _ in range(3))
        self.ws = _lib.workspace(max(L.saix_crc32_workspace_bytes(total), L.saix_index_unpack_workspace_bytes(n)))
        self.units = n
        self.h2d = total
        self.d2h = total + 13 * n
        self.step_device()
        assert bytes(self.blob[-8:].cpu().numpy()) == bytes(self.ist.pack_index(self.eng)[-8:].cpu().numpy())
        self.result = None
        self.config = {"workload": "store: .saix save + load of the index of a 2^26-base random ACGT text "
                                   "(gen_random seed 21 + rank); file image 17n+48 bytes",
                       "bases": n, "file_bytes": total}

    def step_device(self):
        from paper_1404_3448_b200 import _lib
        L, n, s = self.L, self.N, _lib.stream_ptr()
        _lib.check(L.saix_index_pack(_lib.ptr(self.ix.text.t), _lib.ptr(self.ix.sa), _lib.ptr(self.lcp), n, 4, 0,
                                     _lib.ptr(self.blob), _lib.ptr(self.ws), self.ws.numel(), s), "saix_index_pack")
        _lib.check(L.saix_index_unpack(_lib.ptr(self.blob), n, _lib.ptr(self.text_d), _lib.ptr(self.sa_d),
                                       _lib.ptr(self.lcp_d), _lib.ptr(self.isa_d), _lib.ptr(self.ws),
                                       self.ws.numel(), s), "saix_index_unpack")

    def step_e2e(self):
        import io
        sink = io.BytesIO()
        self.ist.save_index(self.eng, sink)
        sink.seek(0)
        self.loaded = self.ist.load_index(sink)

    def extra(self, ms_dev, steps, world):
        return {}

    def cpu_baseline(self):
        import oracle
        n = 1 << 24
        text = self.eng.text.ranks[:n]
        sa, rank = oracle.dc3(text, 4)
        lcp = oracle.lcp(text, sa, rank)
        t0 = time.perf_counter()
        blob = oracle.index_file(text, 4, sa, lcp)
        _, _, sa2, _, lcp2 = oracle.index_load(blob)
        oracle.sparse_build(lcp2)
        dt = time.perf_counter() - t0
        assert np.array_equal(sa2, sa)
        return {"value": n / dt / 1e6, "unit": self.unit, "cores": 1, "kind": "port",
                "sample": f"save (numpy + zlib.crc32) + load (crc check, int64 arrays, rank scatter, sparse-table "
                          f"RMQ rebuild) of a 2^24-base index, single thread ({dt:.1f} s)"}


class Fasta:
    """FASTA ingest (sequence.py:77-157 parse_fasta +
    encode) of a 2^28-base synthetic FASTA (60-column lines, mixed case,
    ~256 records) -- device step: line split, strip, classify, validate,
    concatenate and rank-encode the file bytes resident in HBM; e2e:
    ingest_fasta(bytes) from host memory (H2D of the file inside)."""
    name = "fasta"
    unit = "Mbases/s"
    N = 1 << 28

    def __init__(self, rank: int):
        import torch
        from paper_1404_3448_b200 import _lib
        from paper_1404_3448_b200.fasta import ingest_fasta
        rng = np.random.default_rng(31 + rank)
        lut = np.frombuffer(b"ACGTacgt", np.uint8)
        recs, left, k = [], self.N, 0
        while left > 0:
            m = min(left, 1 << 20)
            seq = lut[rng.integers(0, 8, m)]
            lines = seq[: (m // 60) * 60].reshape(-1, 60)
            body = np.concatenate([lines, np.full((lines.shape[0], 1), 10, np.uint8)], axis=1).ravel().tobytes()
            tail = seq[(m // 60) * 60:].tobytes()
            recs.append(b">chr%d synthetic record %d\n" % (k, k) + body + (tail + b"\n" if tail else b""))
            left -= m
            k += 1
        self.data = b"".join(recs)
        self.dev = _lib.to_device(np.frombuffer(self.data, np.uint8))
        self.ingest = ingest_fasta
        fi = ingest_fasta(self.dev)
        assert fi.total_residues == self.N and len(fi) == k
        self.result = None
        self.units = self.N
        self.h2d = len(self.data)
        self.d2h = 8 * (k + 1) * 2 + sum(len(b">chr%d synthetic record %d" % (i, i)) for i in range(k))
        self.config = {"workload": f"fasta: 2^28-base synthetic FASTA ({len(self.data)} bytes, {k} records, "
                                   "60-column lines, 50% lower case; seed 31 + rank), parse + validate + "
                                   "rank-encode per step", "bases": self.N, "file_bytes": len(self.data)}

    def step_device(self):
        self.ingest(self.dev)

    def step_e2e(self):
        self.ingest(self.data)

    def extra(self, ms_dev, steps, world):
        return {"file_GBps": round(len(self.data) * steps / (ms_dev * 1e-3) / 1e9, 1)}

    def cpu_baseline(self):
        import oracle
        sample = self.data[: 1 << 26]
        sample = sample[: sample.rfind(b"\n") + 1]
        t0 = time.perf_counter()
        recs, err = oracle.fasta(sample, as_ranks=True)
        dt = time.perf_counter() - t0
        assert err is None
        nb = sum(len(r[1]) for r in recs)
        return {"value": nb / dt / 1e6, "unit": self.unit, "cores": 1, "kind": "port",
                "sample": f"first 64 MiB of the file ({nb} bases), oracle_fasta (C restatement of parse_fasta + "
                          f"encode), single thread ({dt:.2f} s)"}


class Cartesian:
    """the Cartesian-tree RMQ engine (rmq.py:61-251)
    built over the LCP array of a 2^26 random text -- device step: tree
    (nearest-value links), Euler tour, ±1 blocks / types / in-block tables,
    block-minimum sparse table, then 10^7 LCA-form range-minimum queries."""
    name = "cartesian"
    unit = "Mbases/s"
    N = 1 << 26
    Q = 10_000_000

    def __init__(self, rank: int):
        import torch
        from paper_1404_3448_b200 import _lib
        from paper_1404_3448_b200.rmq import DeviceSparseTable
        from paper_1404_3448_b200.sequence import gen_random
        from paper_1404_3448_b200.suffix_index import SuffixIndexer
        n = self.N
        self.ranks = encode_ascii(gen_random(n, 1 + rank).residues)
        self.ix = SuffixIndexer(n, 4)
        self.ix.stage(self.ranks)
        self.ix.run_staged()
        self.L = L = _lib.load()
        i32 = lambda k: _lib.empty(k, torch.int32)  # noqa: E731
        self.parent, self.left, self.right, self.first = (i32(n) for _ in range(4))
        self.nodes, self.depths = i32(2 * n - 1), i32(2 * n - 1)
        self.ws = _lib.workspace(L.saix_cartesian_workspace_bytes(n))
        m = 2 * n - 1
        self.b = b = max(1, (m.bit_length() - 1) // 2)
        self.nblocks = (m + b - 1) // b
        self.bargmin, self.bmin, self.types = (i32(self.nblocks) for _ in range(3))
        ncodes = 1 << (b - 1)
        self.present = _lib.empty(((ncodes + 3) & ~3) + 4, torch.uint8)
        self.tab = _lib.empty(ncodes * b * b, torch.uint8)
        self.root = np.zeros(1, np.int64)
        self.bad = np.zeros(1, np.int32)
        rng = np.random.default_rng(2027 + rank)
        self.qi = _lib.to_device(rng.integers(0, n, self.Q))
        self.qj = _lib.to_device(rng.integers(0, n, self.Q))
        self.mlo, self.mhi = _lib.empty(self.Q, torch.int64), _lib.empty(self.Q, torch.int64)
        self.cand = i32(3 * self.Q)
        self.out = _lib.empty(self.Q, torch.int64)
        self.st = None
        self.hlcp = self.ix.lcp[:n].cpu().pin_memory()
        self.hout = torch.empty(self.Q, dtype=torch.int64, pin_memory=True)
        self.step_device()
        self.units = n
        self.h2d = 4 * n
        self.d2h = 8 * self.Q
        self.result = None
        self.config = {"workload": "cartesian: CartesianRmq build (tree + Euler tour + ±1 structure + block sparse "
                                   "table) over the LCP array of a 2^26 random text (gen_random seed 1 + rank) and "
                                   "10^7 LCA-form queries per step", "n": n, "queries": self.Q, "block": b}

    def step_device(self):
        from paper_1404_3448_b200 import _lib
        from paper_1404_3448_b200.rmq import DeviceSparseTable
        L, n, s = self.L, self.N, _lib.stream_ptr()
        _lib.check(L.saix_cartesian_build(_lib.ptr(self.ix.lcp), 4, n, _lib.ptr(self.parent), _lib.ptr(self.left),
                                          _lib.ptr(self.right), _lib.ptr(self.nodes), _lib.ptr(self.depths),
                                          _lib.ptr(self.first), self.root.ctypes.data, _lib.ptr(self.ws),
                                          self.ws.numel(), s), "saix_cartesian_build")
        _lib.check(L.saix_pm1_build(_lib.ptr(self.depths), 2 * n - 1, self.b, _lib.ptr(self.bargmin),
                                    _lib.ptr(self.bmin), _lib.ptr(self.types), _lib.ptr(self.present),
                                    _lib.ptr(self.tab), self.bad.ctypes.data, s), "saix_pm1_build")
        if self.st is None:
            self.st = DeviceSparseTable(self.bmin, 4, self.nblocks)
        else:
            self.st.rebuild()
        _lib.check(L.saix_pm1_query_begin(self.b, _lib.ptr(self.types), _lib.ptr(self.tab), _lib.ptr(self.first),
                                          _lib.ptr(self.qi), _lib.ptr(self.qj), self.Q, _lib.ptr(self.mlo),
                                          _lib.ptr(self.mhi), _lib.ptr(self.cand), s), "saix_pm1_query_begin")
        mid, _ = self.st.query_device(self.mlo, self.mhi)
        _lib.check(L.saix_pm1_query_end(_lib.ptr(self.depths), self.b, _lib.ptr(self.bargmin), _lib.ptr(mid),
                                        _lib.ptr(self.cand), _lib.ptr(self.nodes), self.Q, _lib.ptr(self.out), s),
                   "saix_pm1_query_end")

    def step_e2e(self):
        import torch
        self.ix.lcp.copy_(self.hlcp, non_blocking=True)  # LCP values in from pinned host memory
        self.step_device()
        self.hout.copy_(self.out, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    def extra(self, ms_dev, steps, world):
        return {"queries_per_s": round(self.Q * steps * world / (ms_dev * 1e-3), 1)}

    def cpu_baseline(self):
        import oracle
        from paper_1404_3448_b200.rmq import SparseTable
        lcp = self.ix.lcp[: self.N].cpu().numpy().view(np.uint32).astype(np.int64)
        # parity: the LCA answers for the first 10^5 queries equal the sparse-table argmins
        qi, qj = self.qi[:100_000].cpu().numpy(), self.qj[:100_000].cpu().numpy()
        assert np.array_equal(self.out[:100_000].cpu().numpy(), oracle.argmin_blocked(lcp, qi, qj))
        m = 1 << 24
        t0 = time.perf_counter()
        oracle.cartesian(lcp[:m])
        dt = time.perf_counter() - t0
        return {"value": m / dt / 1e6, "unit": self.unit, "cores": 1, "kind": "port",
                "sample": f"build_cartesian + euler_tour (C port of rmq.py:91-152) over the first 2^24 LCP values, "
                          f"single thread ({dt:.2f} s; the ±1 structure not included); GPU LCA answers matched the "
                          "argmin oracle on 10^5 queries"}


WORKLOADS = {"c2": C2, "c3": C3, "c4": C4, "c5": C5, "store": Store, "fasta": Fasta, "cartesian": Cartesian}


def run_reference(args, rank):
    """Reference algorithm (C oracle port) on the host, same metric/config."""
    import oracle
    if args.workload != "c2":
        print(json.dumps({"impl": "reference", "unavailable": f"workload {args.workload} not wired for the CPU arm"}))
        return
    from paper_1404_3448_b200.sequence import gen_random
    a = gen_random(10_000_000, 11).residues.encode()
    b = gen_random(10_000_000, 12).residues.encode()
    n = len(a) + len(b) + 1
    for _ in range(args.warmup):
        oracle.longest_overlap(a, b)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = oracle.longest_overlap(a, b)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = n * args.steps / tot / 1e6
    cb = {"value": value, "unit": "Mbases/s", "cores": 1, "kind": "port",
          "sample": "full C2 pair (2 x 10 Mbp, GSA n=20,000,001) per step, oracle/saix_oracle.c single thread"}
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Mbases/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": {"workload": "C2", "gsa_bases": n, "result": list(res)},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "Mbases/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def bench(args, rank, world, dist):
    import torch

    from paper_1404_3448_b200 import _lib

    dev = torch.device("cuda", torch.cuda.current_device())
    cls = WORKLOADS[args.workload]
    wl = cls(rank, world, dist) if cls is C4 else cls(rank)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()

    def barrier():
        if dist is not None:
            dist.barrier()

    def timed(step_fn, k):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        barrier()
        torch.cuda.synchronize()
        for e0, e1 in evs:
            flush.zero_()                          # L2 flushed between timed steps (outside events)
            e0.record(st)
            step_fn()
            e1.record(st)
        torch.cuda.synchronize()
        barrier()
        ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
        if dist is not None:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # the section 8(d) model is the reference recursion's level trace: one
    # untimed step with the level-0 window naming off records it
    ref_trace = None
    if args.workload in ("c2", "c3", "c4"):
        prev = _lib.load().saix_dc3_set_window_naming(0)
        wl.step_device()
        torch.cuda.synchronize()
        ref_trace = _lib.dc3_trace()
        _lib.load().saix_dc3_set_window_naming(prev)
    for _ in range(args.warmup):
        wl.step_device()
        wl.step_e2e()
    torch.cuda.synchronize()

    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    ms_dev = timed(wl.step_device, args.steps)    # value: inputs resident in HBM
    ms_e2e = timed(wl.step_e2e, args.steps)       # e2e: pinned host in, results out
    clk = clocks.stop()
    # per-kernel CUDA events (launching stream) in a separate pass of the same
    # K steps, so the timed value carries no event overhead
    prof = []
    if not args.no_prof:
        _lib.prof_enable(True)
        ms_prof = timed(wl.step_device, args.steps)
        prof = _lib.prof_collect()
        _lib.prof_enable(False)
    trace = _lib.dc3_trace()

    launches_per_step = count_our_launches(wl.step_device)
    peak, peak_kind = measured_peak_gbs()
    dom = max(prof, key=lambda e: e["ms"]) if prof else None
    roof = None
    if dom:
        per_launch_ms = dom["ms"] / dom["launches"]
        per_launch_bytes = dom["bytes"] / dom["launches"]
        ach = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": dom["name"], "achieved": round(ach, 1), "peak": peak,
                "peak_source": peak_kind, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": ncu_traffic(args.workload, dom["name"]),
                "bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
                "share_of_step": round(dom["ms"] / ms_dev, 4) if ms_dev else None}
    stage = {e["name"]: round(e["ms"] / args.steps, 4) for e in sorted(prof, key=lambda e: -e["ms"])}
    # whole-DC3 roofline against the section 8(d) contract bytes of the last
    # DC3 level trace (per DC3 call; C4 runs one DC3 per wave)
    dc3_roof = None
    dc3_ms = sum(e["ms"] for e in prof if e["name"].startswith("dc3.")) / args.steps
    if trace and dc3_ms > 0:
        calls = getattr(wl, "dc3_calls_per_step", 1)
        model_trace = ref_trace or trace
        mb = dc3_model_bytes(model_trace) * calls
        ach = mb / (dc3_ms * 1e-3) / 1e9
        dc3_roof = {"model_bytes_per_step": mb, "dc3_ms_per_step": round(dc3_ms, 4),
                    "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                    "levels": [list(t) for t in model_trace], "executed_levels": [list(t) for t in trace],
                    "executed_model_bytes": dc3_model_bytes(trace) * calls,
                    "note": "SURVEY.md 8(d) textbook stage model over the reference recursion's level trace "
                            "(recorded by one untimed step with the level-0 window naming off); "
                            "executed_levels = what this implementation ran"}

    scale = 1e6 if wl.unit == "Mbases/s" else 1.0
    total = getattr(wl, "units_total", wl.units * world)
    value = total * args.steps / (ms_dev * 1e-3) / scale
    e2e_value = total * args.steps / (ms_e2e * 1e-3) / scale

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = wl.cpu_baseline()

    results = wl.result
    if dist is not None and wl.result is not None:
        t = torch.tensor(wl.result, device=dev, dtype=torch.int64)
        allr = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allr, t)
        results = [[int(x) for x in r.tolist()] for r in allr]

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": wl.unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_dev / args.steps, 4),
            "higher_is_better": True, "scaling": getattr(wl, "scaling", "weak"), "vs_baseline": None,
            "dtype": "u32", "data": "synthetic",
            "config": dict(wl.config, l2="flushed between timed steps (512 MiB write)",
                           parallelism=(f"pairs sharded x{world}" if getattr(wl, "scaling", "") == "strong"
                                        else f"replicas x{world}")),
            **wl.extra(ms_dev, args.steps, world),
            "e2e": {"value": round(e2e_value, 2), "unit": wl.unit, "h2d_bytes_per_step": wl.h2d,
                    "d2h_bytes_per_step": wl.d2h, "ms_per_step": round(ms_e2e / args.steps, 4)},
            "gpu_launches": launches_per_step * args.steps,
            "roofline": roof, "dc3_roofline": dc3_roof, "cpu_baseline": cpu, "clocks": clk,
            "stage_ms_per_step": stage,
        }
        if results is not None:
            line["result"] = results
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prof", action="store_true", help="time without per-kernel events")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_env()

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, rank)
        return

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        bench(args, rank, world, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
