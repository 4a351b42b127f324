"""Benchmark of the north-star path: end-to-end spectral clustering
(kNN exp_decay graph -> Lanczos -> k-means) on BASELINE.json's configs[1]
workload (synthetic blobs N=1M, d=64, kNN=32, k=100) on one B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c1]
    python bench.py --impl reference ...   # CPU reference arm (oracle port)

One JSON line on rank 0.  ``value`` = seconds per clustering with X already
resident in HBM (CUDA events around each step, max over ranks);
``e2e`` = the same through the public ``run()`` with host numpy input
(H2D of X and D2H of the report inside the timed region).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "end-to-end clustering sec (N pts, d, k clusters) + per-stage SpMV GB/s, k-means iters/s"
WORKLOADS = {
    # name: (n, d, knn, k, center_scale)
    "c1": (20_000, 32, 16, 20, 1.0),
    "c2": (1_000_000, 64, 32, 100, 0.7),
}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sust=d.get("bf16_tflops_sustained"),
                    src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sust=1400.0, src="fallback")


def make_blobs(n, d, k, cs, seed=0):
    rng = np.random.default_rng(seed)
    centers = rng.normal(0.0, cs, (k, d))
    y = rng.integers(0, k, n)
    x = centers[y] + rng.standard_normal((n, d))
    return np.ascontiguousarray(x), y


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def cpu_reference(n, d, knn, k, cs, sample_n, steps, warmup):
    """Time the CPU oracle (a port of the reference's algorithm) on a bounded
    sample of the workload and extrapolate each stage to full size:
    graph ~ N^2 (all-pairs scan), eigen and k-means ~ N (same iteration
    counts assumed)."""
    from oracle import speclust_oracle as orc

    x, _ = make_blobs(sample_n, d, k, cs, seed=0)
    sigma = float(np.sqrt(d))
    times = []
    stages = None
    for it in range(warmup + steps):
        tm = {}
        t0 = time.perf_counter()
        orc.run_points(x, knn, sigma, k, timings=tm)
        wall = time.perf_counter() - t0
        if it >= warmup:
            times.append(wall)
            stages = tm
    r = n / sample_n
    est = stages["graph"] * r * r + (stages["degrees"] + stages["eigen"] + stages["kmeans"] + stages["metrics"]) * r
    sample = (f"oracle run_points on N={sample_n} (d={d}, kNN={knn}, k={k}); median wall "
              f"{np.median(times):.2f}s; stages {{{', '.join(f'{a}: {b:.2f}' for a, b in stages.items())}}} s; "
              f"extrapolated to N={n}: graph x(N/n)^2, other stages x(N/n)")
    return est, sample, stages


def run_reference_arm(args, wl):
    n, d, knn, k, cs = wl
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count()
    sample_n = args.ref_sample
    est, sample, _ = cpu_reference(n, d, knn, k, cs, sample_n, args.steps, args.warmup)
    line = {
        "metric": METRIC, "value": est, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": est * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: blobs N={n} d={d} kNN={knn} k={k} (BASELINE.json configs[1])"},
        "impl": "reference",
        "cpu_baseline": {"value": est, "unit": "s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": est, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--ref-sample", type=int, default=8000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the public-API end-to-end timing (ncu runs)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the sharded driver (distributed.run_sharded) even at N=1; it is always used for N>1")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference_arm(args, wl)
        return

    import torch
    import torch.distributed as dist

    import paper_1802_04450_b200 as sc
    from paper_1802_04450_b200 import _native as nat
    from paper_1802_04450_b200.pipeline import run_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # N > 1: one problem sharded over the ranks (strong scaling, SURVEY.md
    # §8(e)); every rank holds the same X
    sharded = world > 1 or args.sharded
    if sharded:
        from paper_1802_04450_b200 import distributed as dsc

        comm, ops = dsc.Comm("cuda"), dsc.CudaOps()

    def barrier():
        if world > 1:
            dist.barrier()

    n, d, knn, k, cs = wl
    x_host, _ = make_blobs(n, d, k, cs, seed=0)
    x_pin = torch.from_numpy(x_host).pin_memory()
    x_dev = x_pin.to("cuda")
    sigma = float(np.sqrt(d))

    def cfg_for(points):
        return sc.PipelineConfig(
            input=sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(sigma), pattern="knn", points=points,
                                 knn=knn),
            k_clusters=k, eigen=sc.LanczosConfig(k=k, seed=0), kmeans=sc.KmeansConfig(k=k, seed=0),
            normalize_rows=True)

    lib = nat.load()

    def device_step():
        # X already resident in HBM: the CUDA tensor goes straight to the engine
        if sharded:
            rep = dsc.run_sharded(cfg_for(x_dev), comm, ops)
            return rep, dsc.last_info["nnz"]
        rep, w = run_device(cfg_for(x_dev))
        return rep, w.nnz

    for _ in range(args.warmup):
        device_step()
    torch.cuda.synchronize()

    lib.sc_profile_reset()
    lib.sc_profile_enable(1)
    lib.sc_launch_count_reset()
    times = []
    reports = []
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rep, nnz = device_step()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
            reports.append((rep, nnz))
    barrier()
    torch.cuda.synchronize()
    launches = int(lib.sc_launch_count())
    lib.sc_profile_enable(0)

    def prof(name):
        ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
        lib.sc_profile_query(name.encode(), nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
        return ms.value / max(1, args.steps), cnt.value / max(1, args.steps), work.value / max(1, args.steps)

    kernel_classes = ["knn_order", "knn_tile", "knn_recheck", "knn_fallback", "knn_union", "spmv", "reorth", "ritz", "symeig",
                      "embed", "kmeanspp", "kmeans_assign", "kmeans_update", "ncut"]
    kstats = {c: prof(c) for c in kernel_classes}
    # per step: max over ranks; reported value: median over the timed steps
    t_local = torch.tensor(times, dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    step_max = float(np.median(t_local.cpu().numpy()))

    # ---- end-to-end through the public API: X from pinned host memory is
    # copied to the device inside the timed region, the report (labels,
    # centroids, eigenpairs) comes back to the host
    e2e_times = []
    for _ in range(0 if args.no_e2e else args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep_h = dsc.run_sharded(cfg_for(x_pin), comm, ops) if sharded else sc.run(cfg_for(x_pin))
        _ = rep_h.labeling.labels.sum()
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = float(np.median(e2e_times)) if e2e_times else None

    rep, nnz = reports[-1]
    pk = peaks()
    # dominant kernel class by device time
    dom = max(kstats, key=lambda c: kstats[c][0])
    dms, dlaunch, dwork = kstats[dom]
    tensor_like = dom in ("knn_tile", "kmeans_assign", "ritz")
    if tensor_like:
        achieved = dwork / (dms / 1e3) / 1e12 if dms > 0 else 0.0
        roof = {"bound": "tensor", "achieved": achieved, "peak": pk["bf16"], "unit": "TFLOP/s",
                "frac": achieved / pk["bf16"], "traffic": None, "kernel": dom,
                "peak_src": f"{pk['src']} bf16 burst", "ms_per_step": dms}
    else:
        achieved = dwork / (dms / 1e3) / 1e9 if dms > 0 else 0.0
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm"], "unit": "GB/s",
                "frac": achieved / pk["hbm"], "traffic": None, "kernel": dom, "peak_src": pk["src"],
                "ms_per_step": dms}
    # DRAM traffic of the dominant kernel from the committed ncu capture
    tr = ROOT / "profiles" / "roofline_traffic.json"
    if tr.exists():
        ent = json.loads(tr.read_text()).get(dom)
        if ent:
            roof["traffic"] = ent["bytes"]
            roof["traffic_src"] = ent["capture"]
    spmv_ms, spmv_n, spmv_bytes = kstats["spmv"]
    spmv_gbs = spmv_bytes / (spmv_ms / 1e3) / 1e9 if spmv_ms > 0 else None
    km_iters = rep.labeling.iters_run
    km_s = rep.timings.get("kmeans", 0.0)
    line = {
        "metric": METRIC, "value": step_max, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_max * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: blobs N={n} d={d} kNN={knn} k={k} cs={cs} (BASELINE.json configs[1])",
                   "inputs": "X resident in HBM (512 MB > L2) between steps", "parallelism":
                   f"sharded x{world} (query tiles / row blocks / point shards, NCCL)" if sharded else "single-gpu",
                   "nnz": nnz},
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(x_host.nbytes),
                "d2h_bytes_per_step": int(rep.labeling.labels.nbytes + rep.labeling.centroids.nbytes + 8 * n)},
        "gpu_launches": launches // max(1, args.steps) * args.steps,
        "roofline": roof,
        "stages_s": {kk: round(v, 4) for kk, v in rep.timings.items()},
        "spmv_gbs": spmv_gbs, "spmv_frac_hbm": (spmv_gbs / pk["hbm"]) if spmv_gbs else None,
        "kmeans_iters_per_s": km_iters / km_s if km_s > 0 else None,
        "kmeans_iters": km_iters,
        "kernels_ms_per_step": {c: round(v[0], 3) for c, v in kstats.items() if v[0] > 0},
        "step_times_s": [round(t, 4) for t in times],
        "eigen": {kk: v for kk, v in (dsc.last_info if sharded else __import__(
            "paper_1802_04450_b200.pipeline", fromlist=["x"]).last_info).get("eigen", {}).items() if kk != "history"},
    }
    clk = clocks.summary()
    line["clocks"] = clk
    if rank == 0 and not args.no_cpu_baseline:
        est, sample, _ = cpu_reference(n, d, knn, k, cs, args.ref_sample, 1, 0)
        line["cpu_baseline"] = {"value": est, "unit": "s", "cores": 1, "kind": "port", "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
