"""Per-source-line values of one column of an ncu report's source page
(e.g. "L1 Wavefronts Shared Excessive"):
python tools/ncu_lines_col.py REPORT.ncu-rep "COLUMN" [top]"""
import csv
import subprocess
import sys

rep, col = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
if col not in hdr:
    print("columns:", [h for h in hdr if "avefront" in h or "Shared" in h or "Bank" in h])
    sys.exit(0)
ic = hdr.index(col)
out = []
for r in rows[rows.index(hdr) + 1:]:
    if r and r[0] and not r[0][0].isdigit():
        break  # the next table (SASS)
    if r and r[0] and len(r) > ic:
        try:
            out.append((float((r[ic] or "0").replace(",", "")), int(r[0]), r[1][:110]))
        except ValueError:
            pass
tot = sum(v for v, _, _ in out) or 1
print(f"{col}: total {tot:.0f}")
for v, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{v:14.0f} {100 * v / tot:5.1f}%  L{ln}: {src.strip()}")
