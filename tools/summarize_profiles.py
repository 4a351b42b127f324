"""Summarise a round's ncu captures (gpurun_out/) into profiles/:
  * launch list of one bench step -> per-kernel time share (csv)
  * --set full reports -> key counters per kernel (json)
python tools/summarize_profiles.py <tag>"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"


def launches():
    lines = [ln for ln in (OUT / "launches_c2.csv").read_text().splitlines() if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        per[name][0] += 1
        per[name][1] += float(r["Metric Value"]) / 1e6  # ns -> ms
    total = sum(v[1] for v in per.values())
    # the capture covers several pipeline runs of identical work (warm-up,
    # timed, profiled): one knn_cand_tc2 launch per run
    runs = max(1, sum(c for nm, (c, _) in per.items() if "knn_cand_tc2" in nm))
    out = PROF / f"{tag}_launches_c2_by_kernel.csv"
    with out.open("w") as f:
        f.write("kernel,launches_per_step,ms_per_step,share\n")
        for name, (cnt, ms) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            f.write(f"\"{name}\",{cnt / runs:.0f},{ms / runs:.3f},{ms / total:.4f}\n")
    print(f"wrote {out}: {len(rows)} launches over {runs} runs, {total / runs:.1f} ms of kernels per run")


KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
}


def report(path):
    txt = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")][:120]}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            d[KEYS[h]] = f"{v} {u}".strip()
    return d


launches()
summ = {}
for p in sorted(OUT.glob("*.ncu-rep")):
    try:
        summ[p.stem] = report(p)
    except Exception as e:  # noqa: BLE001
        summ[p.stem] = {"error": str(e)}
(PROF / f"{tag}_ncu_full_summary.json").write_text(json.dumps(summ, indent=1))
print(json.dumps(summ, indent=1))
