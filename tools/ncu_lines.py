"""Per-source-line hot spots of one kernel in an ncu report:
python tools/ncu_lines.py REPORT.ncu-rep [units] [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
iS = hdr.index("Warp Stall Sampling (All Samples)")
iI = hdr.index("Instructions Executed")
out = []
for r in rows[rows.index(hdr) + 1:]:
    if r and r[0]:
        try:
            out.append((int(r[iS]), int(r[iI]), int(r[0]), r[1][:100]))
        except (ValueError, IndexError):
            pass
tot = sum(o[0] for o in out) or 1
toti = sum(o[1] for o in out)
print(f"samples {tot}  warp-instructions {toti} ({toti / units:.0f} per unit)")
for o in sorted(out, reverse=True)[:top]:
    print(f"{o[0]:7d} {100 * o[0] / tot:5.1f}% {o[1] / units:10.0f}/unit  L{o[2]}: {o[3]}")
