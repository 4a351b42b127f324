"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            v = v / 1e6 if u == "ns" else (v / 1e3 if u in ("us", "usecond") else v)
            k = d["Kernel Name"][:70]
            agg[k][0] += 1
            agg[k][1] += v
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:n]:
    print(f"{t:9.2f} ms {c:5d} {k}")
