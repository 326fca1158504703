#!/usr/bin/env python
"""Benchmark of the B200 longest-overlap hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c2|c3|c5|...] [--no-c3]

Default workload (BASELINE.json configs[3], "C4" -- the largest single-GPU
configuration and the one the metric's "pairs/s at 1/2/4/8 B200" is quoted
on): 100,000 synthetic noncoding-like pairs of 2 x 10 kbp
(paper_1404_3448_b200/workloads.py), sharded contiguously across the ranks
(strong scaling); every rank computes longest_overlap for its pairs on the
device and the per-pair results are all-gathered (the path's only
collective).  A "step" is one pass over all 100k pairs.  The same line
carries a "c3" block at N=1: the north star's roofline config (configs[2],
a 2^28 random text, DC3 suffix array + LCP per step, Mbases/s) with the
whole-DC3 roofline against SURVEY.md 8(d)'s contract bytes and against the
bytes this implementation executes.

Other configs: --workload c2 (configs[1], one 2 x 10 Mbp pair), c3, c5
(configs[4], 10^8 sparse-table RMQ queries on a 2^26 text), store, fasta,
cartesian.

--gpus N without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (127.0.0.1 rendezvous).

--impl reference times the reference algorithm on the host -- the C
restatement in oracle/ (kind "port": the reference is pure Python + numba,
nothing to compile) on all host threads -- on the same workload and config:
each step is a bounded sample of the C4 pairs (10,000 pairs, rotating through
the 100k); rank 0 only.
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


def host_info(threads: int) -> dict:
    """CPU model, logical cores and library versions of the host arm."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "threads_used": threads,
            "numpy": np.__version__, "compiler": "gcc -O3 -march=x86-64-v2 (oracle/saix_oracle.c)"}


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
        # parity on ALL 10^8 queries against the leftmost-argmin definition
        # (untimed; block minima + sparse table over them, every host thread)
        lcp = self.ix.lcp[: self.N].cpu().numpy().view(np.uint32).astype(np.int64)
        threads = os.cpu_count() or 1
        got = self.out.cpu().numpy()
        want = oracle.argmin_sparse_blocked(lcp, self.hqi.numpy(), self.hqj.numpy(), threads=threads)
        mism = int(np.count_nonzero(got != want))
        assert mism == 0, f"{mism} of {self.Q} C5 answers differ from the oracle"
        self.parity = {"queries_checked": self.Q, "mismatches": mism}
        del got, want
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
                          f"single thread ({dt:.2f} s); GPU answers matched the argmin oracle on all 10^8 queries"}


def c4_generate(lo: int, hi: int):
    from paper_1404_3448_b200.workloads import c4_generate as gen
    return gen(lo, hi)


C4_TOTAL = 100_000
C4_REF_SAMPLE = 10_000


def c4_config(world: int) -> dict:
    """The C4 `config` object -- identical on both arms."""
    return {"workload": "C4: 100k pairs of 2 x 10 kbp AT-rich random sequences (W = 0.3/0.2/0.2/0.3) with one "
                        "planted shared block of 32..256 bases (paper_1404_3448_b200/workloads.py); "
                        "longest_overlap of every pair per step",
            "pairs": C4_TOTAL, "residues_per_pair": 20_000,
            "l2": "inputs (2 GB) larger than L2; L2 also flushed between timed steps (512 MiB write)",
            "parallelism": f"pairs sharded x{world}"}


class C4:
    """configs[3]: 100k synthetic 10 kbp noncoding-like pairs (workloads.py),
    sharded contiguously across ranks (strong scaling); the per-pair results
    are all-gathered to every rank over NCCL inside the step (the one
    collective of the path)."""
    name = "c4"
    unit = "pairs/s"
    scaling = "strong"
    TOTAL = C4_TOTAL

    def __init__(self, rank: int, world: int = 1, dist=None):
        import torch

        import paper_1404_3448_b200 as sx
        from paper_1404_3448_b200.workloads import shard
        self.lo, self.hi = shard(self.TOTAL, world, rank)
        self.seqs, self.offs = c4_generate(self.lo, self.hi)
        self.P = self.hi - self.lo
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
        self.config = c4_config(world)
        self.dc3_calls_per_step = getattr(self.ob, "dc3_calls", len(self.ob.waves))

    def _gather(self):
        if self.dist is None or self.world == 1:
            return
        from paper_1404_3448_b200.distributed import NcclComm, gather_results, gather_results_nccl
        if self.dist.get_backend() == "nccl":   # the library's own NCCL communicator
            if getattr(self, "comm", None) is None:
                self.comm = NcclComm(self.dist, self.world, self.dist.get_rank())
            self.full = gather_results_nccl(self.ob.out[: 3 * self.P], self.TOTAL, self.world, self.comm)
        else:
            self.full = gather_results(self.ob.out[: 3 * self.P], self.TOTAL, self.world, self.dist)

    def step_device(self):
        self.ob.run_device()
        self._gather()

    def step_e2e(self):
        import torch
        self.ob.run_from_host(self.hseqs)     # chunked H2D overlapped with the chunks' pairs
        self._gather()
        self.hout.copy_(self.ob.out[: 3 * self.P], non_blocking=True)
        torch.cuda.current_stream().synchronize()

    def extra(self, ms_dev, steps, world):
        return {}

    def cpu_baseline(self):
        """The oracle on every host thread over ALL of this rank's pairs
        (100k at N=1): timed, and every GPU answer compared."""
        import oracle
        threads = os.cpu_count() or 1
        t0 = time.perf_counter()
        want = oracle.overlap_batch(self.seqs, self.offs, threads=threads)
        dt = time.perf_counter() - t0
        got = self.ob.results()
        mism = int(np.count_nonzero(np.any(got != want, axis=1)))
        assert mism == 0, f"{mism} of {self.P} C4 pairs differ from the oracle"
        self.parity = {"pairs_checked": int(self.P), "mismatches": mism}
        return {"value": self.P / dt, "unit": self.unit, "cores": threads, "kind": "port",
                "sample": f"all {self.P} C4 pairs, oracle/saix_oracle.c (C restatement of overlap.py:110-152 + "
                          f"suffix_index.py DC3/Kasai) on {threads} host threads ({dt:.1f} s); GPU answers matched "
                          "on every pair", "host": host_info(threads)}


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
    """Reference algorithm (C oracle port, all host threads) on the host, same
    metric/config as our arm; each step is a bounded sample of the workload."""
    import oracle
    threads = os.cpu_count() or 1
    common = {"impl": "reference", "metric": METRIC, "n_gpus": args.gpus, "steps": args.steps,
              "warmup": args.warmup, "higher_is_better": True, "vs_baseline": None, "dtype": "u32",
              "data": "synthetic"}
    if args.workload == "c4":
        nsteps = args.warmup + args.steps
        span = min(C4_TOTAL, nsteps * C4_REF_SAMPLE)
        seqs, offs = c4_generate(0, span)
        times = []
        for k in range(nsteps):
            p0 = (k * C4_REF_SAMPLE) % span
            p1 = min(p0 + C4_REF_SAMPLE, span)
            sq = seqs[offs[2 * p0]: offs[2 * p1]]
            of = offs[2 * p0: 2 * p1 + 1] - offs[2 * p0]
            t0 = time.perf_counter()
            oracle.overlap_batch(sq, of, threads=threads)
            if k >= args.warmup:
                times.append((time.perf_counter() - t0, p1 - p0))
        tot = sum(t for t, _ in times)
        pairs = sum(p for _, p in times)
        value = pairs / tot
        sample = (f"{C4_REF_SAMPLE} C4 pairs per step (rotating through the first {span}), "
                  f"oracle/saix_oracle.c on {threads} host threads")
        line = dict(common, value=value, unit="pairs/s", ms_per_step=1e3 * tot / len(times),
                    scaling="strong", config=c4_config(args.gpus))
    elif args.workload == "c2":
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
        threads = 1
        sample = "full C2 pair (2 x 10 Mbp, GSA n=20,000,001) per step, oracle/saix_oracle.c single thread"
        line = dict(common, value=value, unit="Mbases/s", ms_per_step=1e3 * tot / args.steps, scaling="weak",
                    config={"workload": "C2", "gsa_bases": n, "result": list(res)})
    else:
        print(json.dumps({"impl": "reference", "unavailable": f"workload {args.workload} not wired for the CPU arm"}))
        return
    line["cpu_baseline"] = {"value": line["value"], "unit": line["unit"], "cores": threads, "kind": "port",
                            "sample": sample, "host": host_info(threads)}
    line["e2e"] = {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)


def measure(wl, args, rank, world, dist, dev, flush, record_ref_trace=True):
    """Warm up, then time K device-resident steps and K end-to-end steps
    (CUDA events on the launching stream, L2 flushed between steps, barrier +
    synchronize on both sides, max over ranks), one more K-step pass with
    per-kernel events, and the launch count of one step."""
    import torch

    from paper_1404_3448_b200 import _lib
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
    if record_ref_trace and wl.name in ("c2", "c3"):
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
        timed(wl.step_device, args.steps)
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
        tr = ncu_traffic(wl.name, dom["name"])
        roof = {"bound": "hbm", "kernel": dom["name"], "achieved": round(ach, 1), "peak": peak,
                "peak_source": peak_kind, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": tr, "traffic_over_algorithmic": (round(tr / per_launch_bytes, 3)
                                                             if tr and per_launch_bytes else None),
                "bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
                "share_of_step": round(dom["ms"] / ms_dev, 4) if ms_dev else None}
    stage = {e["name"]: round(e["ms"] / args.steps, 4) for e in sorted(prof, key=lambda e: -e["ms"])}
    # whole-DC3 roofline against the section 8(d) contract bytes, both over
    # the reference recursion's level trace and over what actually ran
    dc3_roof = None
    dc3_ms = sum(e["ms"] for e in prof if e["name"].startswith("dc3.")) / args.steps
    model_fn = getattr(wl, "dc3_model", None)
    if model_fn is not None and dc3_ms > 0:
        dc3_roof = model_fn(dc3_ms, peak)
    elif trace and dc3_ms > 0:
        calls = getattr(wl, "dc3_calls_per_step", 1)
        model_trace = ref_trace or trace
        mb = dc3_model_bytes(model_trace) * calls
        xb = dc3_model_bytes(trace) * calls
        ach = mb / (dc3_ms * 1e-3) / 1e9
        dc3_roof = {"model_bytes_per_step": mb, "dc3_ms_per_step": round(dc3_ms, 4),
                    "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                    "executed_model_bytes": xb,
                    "executed_frac": round(xb / (dc3_ms * 1e-3) / 1e9 / peak, 4),
                    "levels": [list(t) for t in model_trace], "executed_levels": [list(t) for t in trace],
                    "note": "frac: SURVEY.md 8(d) textbook stage model over the reference recursion's level trace "
                            "(recorded by one untimed step with the level-0 window naming off) / DC3 time; "
                            "executed_frac: the same model over the levels this implementation ran"}

    scale = 1e6 if wl.unit == "Mbases/s" else 1.0
    total = getattr(wl, "units_total", wl.units * world)
    return {"value": total * args.steps / (ms_dev * 1e-3) / scale, "ms_dev": ms_dev,
            "e2e_value": total * args.steps / (ms_e2e * 1e-3) / scale, "ms_e2e": ms_e2e,
            "roofline": roof, "dc3_roofline": dc3_roof, "stage": stage, "clocks": clk,
            "gpu_launches": launches_per_step * args.steps}


def c3_block(args, dev, flush):
    """The north star's roofline config (C3) measured in the same run: a 2^28
    DC3 suffix array + LCP per step, N=1 only."""
    wl = C3(0)
    m = measure(wl, args, 0, 1, None, dev, flush)
    blk = {"workload": wl.config["workload"], "value": round(m["value"], 2), "unit": wl.unit,
           "ms_per_step": round(m["ms_dev"] / args.steps, 4),
           "e2e": {"value": round(m["e2e_value"], 2), "unit": wl.unit, "h2d_bytes_per_step": wl.h2d,
                   "d2h_bytes_per_step": wl.d2h, "ms_per_step": round(m["ms_e2e"] / args.steps, 4)},
           "gpu_launches": m["gpu_launches"], "roofline": m["roofline"], "dc3_roofline": m["dc3_roofline"],
           "clocks": m["clocks"], "stage_ms_per_step": m["stage"]}
    if not args.no_cpu_baseline:
        blk["cpu_baseline"] = wl.cpu_baseline()
    del wl
    return blk


def bench(args, rank, world, dist):
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    cls = WORKLOADS[args.workload]
    wl = cls(rank, world, dist) if cls is C4 else cls(rank)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    m = measure(wl, args, rank, world, dist, dev, flush)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = wl.cpu_baseline()

    results = wl.result
    if dist is not None and wl.result is not None:
        t = torch.tensor(wl.result, device=dev, dtype=torch.int64)
        allr = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allr, t)
        results = [[int(x) for x in r.tolist()] for r in allr]

    c3 = None
    if args.workload == "c4" and world == 1 and not args.no_c3:
        del wl.ob
        torch.cuda.empty_cache()
        c3 = c3_block(args, dev, flush)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(m["value"], 2), "unit": wl.unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(m["ms_dev"] / args.steps, 4),
            "higher_is_better": True, "scaling": getattr(wl, "scaling", "weak"), "vs_baseline": None,
            "dtype": "u32", "data": "synthetic",
            "config": dict(wl.config) if wl.name == "c4" else dict(
                wl.config, l2="flushed between timed steps (512 MiB write)", parallelism=f"replicas x{world}"),
            **wl.extra(m["ms_dev"], args.steps, world),
            "e2e": {"value": round(m["e2e_value"], 2), "unit": wl.unit, "h2d_bytes_per_step": wl.h2d,
                    "d2h_bytes_per_step": wl.d2h, "ms_per_step": round(m["ms_e2e"] / args.steps, 4)},
            "gpu_launches": m["gpu_launches"],
            "roofline": m["roofline"], "dc3_roofline": m["dc3_roofline"], "cpu_baseline": cpu, "clocks": m["clocks"],
            "stage_ms_per_step": m["stage"],
        }
        roof = m["roofline"]
        if wl.name == "c4" and roof and roof.get("kernel") == "pairs.dc3_onchip":
            # the pair DC3 works out of shared memory (HBM moves only its input,
            # roofline.traffic): the same model bytes against the aggregate
            # shared-memory bandwidth, 128 B/clk per SM at the sampled SM clock
            mhz = (m["clocks"] or {}).get("sm_mhz") or 1965.0
            smem_peak = 128.0 * 148 * mhz * 1e6 / 1e9
            line["onchip_roofline"] = {"bound": "smem", "kernel": roof["kernel"], "achieved": roof["achieved"],
                                       "peak": round(smem_peak, 1), "unit": "GB/s",
                                       "frac": round(roof["achieved"] / smem_peak, 4),
                                       "peak_source": f"128 B/clk/SM x 148 SMs x {mhz:.0f} MHz"}
        if getattr(args, "shared_devices", 0):
            line["config"]["shared_devices"] = (f"{world} ranks on {args.shared_devices} GPU(s) over gloo: "
                                                "validates the sharded path, not a scaling number")
        if getattr(wl, "parity", None):
            line["parity"] = wl.parity
        if results is not None:
            line["result"] = results
        if c3 is not None:
            line["c3"] = c3
        print(json.dumps(line), flush=True)


def relaunch_under_torchrun(args) -> int:
    """`--gpus N` without a torchrun environment: run N ranks of this script
    under torch.distributed.run (one process per GPU, 127.0.0.1)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c4")
    ap.add_argument("--no-c3", action="store_true", help="skip the in-line C3 block of the C4 line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prof", action="store_true", help="time without per-kernel events")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    args.gpus = world

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, rank)
        return

    import torch
    ndev = max(1, torch.cuda.device_count())
    # more ranks than GPUs (a 1-GPU box validating the N-rank path): ranks
    # share devices over gloo and the line says so; timings are not scaling
    args.shared_devices = ndev if world > ndev else 0
    torch.cuda.set_device(local % ndev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.shared_devices:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        bench(args, rank, world, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
