"""Text summary of ncu --set full captures (one line block per kernel):
python tools/full_summary.py REPORT.ncu-rep [...] > profiles/...txt"""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
        "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "L1/TEX Hit Rate", "L2 Hit Rate"]

for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if not rows:
        continue
    hdr = rows[0]
    iname, imetric, iunit, ival = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), \
        hdr.index("Metric Value")
    seen = {}
    kname = None
    for r in rows[1:]:
        kname = r[iname]
        if r[imetric] in KEYS and r[imetric] not in seen:
            seen[r[imetric]] = f"{r[ival]} {r[iunit]}".strip()
    print(f"== {rep.split('/')[-1]}: {kname[:90] if kname else '?'}")
    for k in KEYS:
        if k in seen:
            print(f"   {k:36s} {seen[k]}")
