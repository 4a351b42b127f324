"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, sys
r = list(csv.reader(open(sys.argv[1])))
h = r[1]
rows = r[2:]
S = h.index("Warp Stall Sampling (All Samples)")
E = h.index("Instructions Executed")
tot = sum(float(x[S] or 0) for x in rows)
toti = sum(float(x[E] or 0) for x in rows)
print(f"samples {tot:.0f} warp-instrs {toti:.3g}")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k, x in sorted(enumerate(rows), key=lambda t: -float(t[1][S] or 0))[:n]:
    st = sorted(((float(x[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:2]
    print(f"{k:5d} {float(x[S])/tot*100:5.1f}% ex={float(x[E] or 0):.3g} {x[1].strip()[:60]:60s} {st}")
