"""Summarise an `ncu --csv` launch list: time share, DRAM bytes per kernel."""
import csv, collections, sys

def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]; idx = {k: i for i, k in enumerate(hdr)}
    per = collections.OrderedDict()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
             "ns": 1e-3, "us": 1, "ms": 1e3}
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        d = per.setdefault(r[idx["ID"]], {"name": r[idx["Kernel Name"]]})
        v = float(r[idx["Metric Value"]].replace(",", ""))
        d[r[idx["Metric Name"]]] = v * scale.get(r[idx["Metric Unit"]], 1)
    return per

def main(path, top=25):
    per = load(path)
    agg = collections.defaultdict(lambda: [0.0, 0, 0.0, 0.0])
    tot = 0.0
    for d in per.values():
        t = d.get("gpu__time_duration.sum", 0.0)
        nm = d["name"].split("(")[0].replace("void ", "")[:70]
        a = agg[nm]; a[0] += t; a[1] += 1
        a[2] += d.get("dram__bytes_read.sum", 0.0); a[3] += d.get("dram__bytes_write.sum", 0.0)
        tot += t
    print(f"total {tot:.1f} us over {len(per)} launches")
    print(f"{'us':>9} {'n':>4} {'share':>6} {'DRAM MB':>9} {'GB/s':>7}  kernel")
    for nm, (t, c, r, w) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{t:9.1f} {c:4d} {100*t/tot:5.1f}% {(r+w)/1e6:9.1f} {(r+w)/t/1e3 if t else 0:7.0f}  {nm}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
