"""Per-kernel summary of one C2 run from an ncu launch list
(--metrics gpu__time_duration.sum --csv): the launches between the first two
knn_prep_f16 kernels (one whole pipeline run) grouped by kernel name."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
data = rows[1:]
names = [r[4].split("(")[0].replace("void ", "").replace("sc::", "").replace("<unnamed>::", "") for r in data]
dur = [float(r[-1]) for r in data]
starts = [i for i, nm in enumerate(names) if "knn_prep_f16" in nm]
a, b = starts[0], starts[1] if len(starts) > 1 else len(names)
agg, cnt = collections.Counter(), collections.Counter()
for nm, d in zip(names[a:b], dur[a:b]):
    agg[nm] += d
    cnt[nm] += 1
tot = sum(agg.values())
w = csv.writer(sys.stdout)
w.writerow(["kernel", "launches", "total_ms", "share", "mean_us"])
for nm, d in agg.most_common():
    w.writerow([nm, cnt[nm], round(d / 1e6, 3), round(d / tot, 4), round(d / cnt[nm] / 1e3, 2)])
w.writerow(["TOTAL", b - a, round(tot / 1e6, 3), 1.0, ""])
