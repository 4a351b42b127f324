"""Benchmark of the north-star path: end-to-end spectral clustering
(kNN exp_decay graph -> Lanczos -> k-means) on BASELINE.json's configs[1]
workload (synthetic blobs N=1M, d=64, kNN=32, k=100) on one B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c1|c3|c3h]
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
    "c3": (4_000_000, 128, 32, 1000, 1.0),
    "c3h": (1_000_000, 128, 32, 1000, 1.0),
}
CONFIG_NOTE = {"c1": "BASELINE.json configs[0]", "c2": "BASELINE.json configs[1]",
               "c3": "BASELINE.json configs[2] at 1 GPU", "c3h": "BASELINE.json configs[2] shape at N/4"}


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
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region, in-process through NVML (no nvidia-smi subprocess: forking a CUDA
    process every 0.2 s stalled the host-driven Lanczos loop and showed up as
    step-to-step variance); falls back to nvidia-smi if NVML is missing."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, [4 flags])
        self.period = 0.1
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._bits = (pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                          pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap)
        except Exception:
            self._nv = None

    def _sample(self):
        if self._nv is not None:
            nv = self._nv
            sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            return float(sm), float(mx), [bool(r & b) for b in self._bits]
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        parts = [p.strip() for p in out.stdout.strip().split(",")]
        return float(parts[0]), float(parts[1]), [p.lower() == "active" for p in parts[2:6]]

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self._stop.wait(self.period)

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
        reasons = sorted({self.NAMES[i] for s in self.samples for i in range(4) if s[2][i]})
        return {"sm_mhz": float(np.median([s[0] for s in self.samples])),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._nv is not None else "nvidia-smi"}


# ---------------------------------------------------------------------------
def host_cpu():
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def oracle_run(n, d, knn, k, cs, seed=0):
    """One timed CPU-oracle clustering (a numpy port of the reference's
    algorithm, test infrastructure) of the blobs workload; numpy's BLAS uses
    every host core.  Returns (wall seconds, stage seconds, labels, planted)."""
    from oracle import speclust_oracle as orc

    x, y = make_blobs(n, d, k, cs, seed=seed)
    tm = {}
    t0 = time.perf_counter()
    out = orc.run_points(x, knn, float(np.sqrt(d)), k, timings=tm)
    return time.perf_counter() - t0, tm, out["labels"], y


def extrapolate(stages, n, sample_n):
    """Model only (never a measured value): graph ~ N^2 (all-pairs scan), the
    other stages ~ N at the sample's iteration counts."""
    r = n / sample_n
    return stages["graph"] * r * r + sum(v for s, v in stages.items() if s != "graph") * r


def run_reference_arm(args, wl):
    """The reference arm: the CPU oracle timed on a bounded sample of the
    workload (N = --ref-sample points of the same distribution), every step
    measured; ``value`` is that measured sample time.  The full-size
    extrapolation is a separate, labelled estimate."""
    n, d, knn, k, cs = wl
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sn = min(args.ref_sample, n)
    times, stages = [], None
    t_run0 = time.perf_counter()
    for it in range(args.warmup + args.steps):
        wall, tm, _, _ = oracle_run(sn, d, knn, k, cs)
        if it >= args.warmup:
            times.append(wall)
            stages = tm
    run_s = time.perf_counter() - t_run0
    v = float(np.median(times))
    cpu = host_cpu()
    sample = (f"oracle run_points on N={sn} blobs (d={d}, kNN={knn}, k={k}, cs={cs}) per step, measured; "
              f"stages {{{', '.join(f'{a}: {b:.3f}' for a, b in stages.items())}}} s")
    line = {
        "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}-sample: blobs N={sn} d={d} kNN={knn} k={k} cs={cs} "
                               f"(bounded sample of {CONFIG_NOTE[args.workload]}, N={n})",
                   "same_config": sn == n},
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "s", "cores": cpu["nproc"], "kind": "port", "sample": sample,
                         "cpu_model": cpu["model"]},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_times_s": [round(t, 3) for t in times],
        "run_s": round(run_s, 2),
        "estimate_full_s": {"value": extrapolate(stages, n, sn), "n": n,
                            "model": "graph x (N/n)^2, other stages x (N/n); an estimate, not a measurement"},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def syn200_run(torch, sc, run_device):
    """The paper's Syn200 (SBM 200 blocks x 100 nodes, p=0.3, q=0.01, k=200;
    PAPER.md:536-550): eigensolver and k-means seconds beside the paper's
    published K20c CUDA numbers (4.1153 s / 0.02478 s).  The graph comes from
    this engine's device SBM generator (its own Philox stream)."""
    from paper_1802_04450_b200.sbm import SbmConfig, sbm_generate_device

    w, truth = sbm_generate_device(SbmConfig(block_sizes=(100,) * 200, p_in=0.3, p_out=0.01, seed=0))
    cfg = sc.PipelineConfig(input=sc.MatrixInput(matrix=w), k_clusters=200,
                            eigen=sc.LanczosConfig(k=200, seed=0), kmeans=sc.KmeansConfig(k=200, seed=0),
                            normalize_rows=True)
    run_device(cfg)  # warm-up
    reps = []
    for _ in range(3):
        torch.cuda.synchronize()
        rep, _ = run_device(cfg)
        reps.append(rep)
    eig = float(np.median([r.timings["eigen"] for r in reps]))
    km = float(np.median([r.timings["kmeans"] for r in reps]))
    return {"workload": "Syn200: SBM 200 x 100, p=0.3, q=0.01, k=200 (PAPER.md:536-550)", "edges": w.nnz // 2,
            "eigen_s": eig, "kmeans_s": km, "paper_k20c_eigen_s": 4.1153, "paper_k20c_kmeans_s": 0.02478,
            "eigen_speedup_vs_paper": 4.1153 / eig, "kmeans_speedup_vs_paper": 0.02478 / km,
            "ari_vs_planted": float(sc.adjusted_rand_index(reps[-1].labeling.labels, truth.cpu().numpy())),
            "note": "paper graph had 773,388 edges (inconsistent with its p, q; BASELINE.md)"}


def c3_run(torch, sc, nat, run_device, lib):
    """One full-size C3 clustering (BASELINE.json configs[2]: blobs N=4M,
    d=128, kNN=32, k=1000, m=2000) on this GPU with X resident in HBM, timed
    with CUDA events and no profiling; plus one profiled Lloyd assignment at
    C3's embedding shape for the tensor-core fraction of the assignment GEMM."""
    from paper_1802_04450_b200 import pipeline as pl

    free, total = torch.cuda.mem_get_info()
    if total < 150e9:
        return {"skipped": f"needs ~150 GB of device memory, this GPU has {total / 1e9:.0f} GB"}
    n, d, knn, k, cs = WORKLOADS["c3"]
    x, y = make_blobs(n, d, k, cs, seed=0)
    xd = torch.from_numpy(x).cuda()
    del x
    cfg = sc.PipelineConfig(
        input=sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))), pattern="knn", points=xd,
                             knn=knn),
        k_clusters=k, eigen=sc.LanczosConfig(k=k, seed=0), kmeans=sc.KmeansConfig(k=k, seed=0), normalize_rows=True)
    lib.sc_profile_enable(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep, w = run_device(cfg)
    e1.record()
    torch.cuda.synchronize()
    secs = e0.elapsed_time(e1) / 1e3
    out = {"workload": f"c3: blobs N={n} d={d} kNN={knn} k={k} cs={cs} (BASELINE.json configs[2]), X resident",
           "seconds": secs, "stages_s": {a: round(b, 3) for a, b in rep.timings.items()}, "nnz": w.nnz,
           "eigen": {a: b for a, b in pl.last_info.get("eigen", {}).items() if a != "history"},
           "kmeans_iters": rep.labeling.iters_run,
           "max_eigen_residual": float(np.max(rep.eigen_residuals)),
           "lambda_1": float(rep.eigenvalues[0]), "lambda_k": float(rep.eigenvalues[-1]),
           "ari_vs_planted": float(sc.adjusted_rand_index(rep.labeling.labels, y))}
    del rep, w, xd, cfg
    nat.load().sc_trim_pool()
    torch.cuda.empty_cache()
    # assignment GEMM at C3's embedding shape (n x k unit rows, k centroids)
    g = torch.Generator(device="cuda").manual_seed(1)
    cen = torch.randn((k, k), generator=g, device="cuda", dtype=torch.float64)
    lab = torch.randint(0, k, (n,), generator=g, device="cuda")
    v = cen[lab] + 0.05 * torch.randn((n, k), generator=g, device="cuda", dtype=torch.float64)
    v /= v.norm(dim=1, keepdim=True)
    # one seed row per planted cluster (what k-means++ finds on this data)
    first = torch.full((k,), n, dtype=torch.int64, device="cuda").scatter_reduce(
        0, lab, torch.arange(n, device="cuda"), reduce="amin")
    init = v[first.clamp(max=n - 1)].contiguous()
    del cen, lab
    km = __import__("paper_1802_04450_b200.kmeans", fromlist=["lloyd_device"])
    lib.sc_profile_reset()
    lib.sc_profile_enable(1)
    km.lloyd_device(v, init, sc.KmeansConfig(k=k, max_iters=2))
    torch.cuda.synchronize()
    lib.sc_profile_enable(0)
    ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
    lib.sc_profile_query(b"kmeans_assign", nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
    pk = peaks()
    tf = work.value / (ms.value / 1e3) / 1e12 if ms.value > 0 else None
    out["assign_gemm"] = {"shape": f"{n} x {k} embedding, {k} centroids", "launches": cnt.value,
                          "ms_per_launch": ms.value / max(1, cnt.value), "tflops": tf,
                          "frac_of_bf16_peak": tf / pk["bf16"] if tf else None}
    del v, init
    nat.load().sc_trim_pool()
    torch.cuda.empty_cache()
    return out


def make_c5(torch, n, d=256, k=10_000, seed=0):
    """C5's embedding (SURVEY.md:594): k Gaussian centres N(0, 1) in d
    dimensions, points = centre + N(0, 0.3^2) noise, rows normalised; drawn
    on the device in fp32 (10 GB at full size) and held in fp64 for Lloyd.
    Init rows = default_rng(0).choice(n, k, replace=False), the reference's
    ``random_points`` init (kmeans.py:203-205)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    cen = torch.randn((k, d), generator=g, device="cuda", dtype=torch.float32)
    lab = torch.randint(0, k, (n,), generator=g, device="cuda")
    v = torch.empty((n, d), dtype=torch.float64, device="cuda")
    step = 1 << 21
    for a in range(0, n, step):
        b = min(n, a + step)
        t = cen[lab[a:b]] + 0.3 * torch.randn((b - a, d), generator=g, device="cuda", dtype=torch.float32)
        t /= t.norm(dim=1, keepdim=True)
        v[a:b] = t
    rows = np.random.default_rng(0).choice(n, size=k, replace=False)
    init = v[torch.from_numpy(rows).to("cuda")].contiguous()
    return v, init, lab


def c5_run(torch, n=10_000_000, iters=20):
    """C5 at full size (BASELINE.json configs[4]: k-means on a 10M x 256
    embedding, k = 10,000): a fixed ``iters`` Lloyd iterations
    (tol_changes = 0, max_iters = iters) timed with CUDA events and no
    profiling, then a second profiled run for the per-kernel rates."""
    import paper_1802_04450_b200 as sc
    from paper_1802_04450_b200 import _native as nat
    from paper_1802_04450_b200.kmeans import lloyd_device

    free, total = torch.cuda.mem_get_info()
    if total < 100e9:
        return {"skipped": f"needs ~60 GB of device memory, this GPU has {total / 1e9:.0f} GB"}
    k, d = 10_000, 256
    lib = nat.load()
    v, init, lab = make_c5(torch, n, d, k)
    cfg = sc.KmeansConfig(k=k, max_iters=iters, init="random_points")
    lib.sc_profile_enable(0)
    lloyd_device(v[: 1 << 16], init[:256].contiguous(), sc.KmeansConfig(k=256, max_iters=2))  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    labels, cent, hist, it = lloyd_device(v, init, cfg)
    e1.record()
    torch.cuda.synchronize()
    secs = e0.elapsed_time(e1) / 1e3
    out = {"workload": f"c5: Lloyd on a {n} x {d} embedding, k={k}, {iters} iterations from random_points "
                       "(BASELINE.json configs[4])",
           "seconds": secs, "iters_run": it, "s_per_iter": secs / max(1, it),
           "sse_first": float(hist[0]), "sse_last": float(hist[-1]),
           "sse_monotone": bool(np.all(np.diff(hist) <= 1e-9 * abs(hist[0]))),
           "ari_vs_planted": float(sc.adjusted_rand_index(labels.cpu().numpy(), lab.cpu().numpy()))}
    del labels, cent
    lib.sc_profile_reset()
    lib.sc_profile_enable(1)
    lloyd_device(v, init, sc.KmeansConfig(k=k, max_iters=3, init="random_points"))
    torch.cuda.synchronize()
    lib.sc_profile_enable(0)
    pk = peaks()
    kern = {}
    for c in ("kmeans_assign", "kmeans_update"):
        ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
        lib.sc_profile_query(c.encode(), nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
        kern[c] = {"launches": cnt.value, "ms_total": round(ms.value, 3), "work": work.value}
    a = kern["kmeans_assign"]
    if a["ms_total"] > 0:
        tf = a["work"] / (a["ms_total"] / 1e3) / 1e12
        a["tflops"] = tf
        a["frac_of_bf16_peak"] = tf / pk["bf16"]
    out["kernels"] = kern
    del v, init, lab
    lib.sc_trim_pool()
    torch.cuda.empty_cache()
    return out


def c4_run(torch):
    """C4 at full size (BASELINE.json configs[3]): a planted-partition graph
    of 500 blocks x 32,000 nodes (p_in 1.6e-3, p_out 8e-7: ~512M undirected
    unit-weight edges, SURVEY.md:594) drawn on this GPU by the device SBM
    generator, then run() on it as MatrixInput with k = 500 (eigensolver +
    k-means).  The 16M x 1001 Krylov basis (128 GB) does not fit beside a
    separate 16M x 500 eigenvector array, so the pipeline keeps the result in
    the basis (eigensolve_device_basis)."""
    import paper_1802_04450_b200 as sc
    from paper_1802_04450_b200 import pipeline as pl
    from paper_1802_04450_b200.sbm import SbmConfig, sbm_generate_device

    free, total = torch.cuda.mem_get_info()
    if total < 170e9:
        return {"skipped": f"needs ~165 GB of device memory, this GPU has {total / 1e9:.0f} GB"}
    t0 = time.perf_counter()
    w, truth = sbm_generate_device(SbmConfig(block_sizes=(32_000,) * 500, p_in=1.6e-3, p_out=8e-7, seed=0))
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    k = 500
    cfg = sc.PipelineConfig(input=sc.MatrixInput(matrix=w), k_clusters=k, eigen=sc.LanczosConfig(k=k, seed=0),
                            kmeans=sc.KmeansConfig(k=k, seed=0), normalize_rows=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep, _ = pl.run_device(cfg)
    e1.record()
    torch.cuda.synchronize()
    out = {"workload": "c4: SBM 500 x 32000 nodes, p_in 1.6e-3, p_out 8e-7, k=500, unit weights "
                       "(BASELINE.json configs[3]), graph resident",
           "n": w.n_rows, "nnz": w.nnz, "generate_s": gen_s, "seconds": e0.elapsed_time(e1) / 1e3,
           "stages_s": {a: round(b, 3) for a, b in rep.timings.items()},
           "eigen": {a: b for a, b in pl.last_info.get("eigen", {}).items() if a != "history"},
           "kmeans_iters": rep.labeling.iters_run, "max_eigen_residual": float(np.max(rep.eigen_residuals)),
           "lambda_1": float(rep.eigenvalues[0]), "lambda_k": float(rep.eigenvalues[-1]),
           "ari_vs_planted": float(sc.adjusted_rand_index(rep.labeling.labels, truth.cpu().numpy())),
           "ncut": float(rep.ncut_value), "warnings": rep.warnings}
    del w, truth, rep
    from paper_1802_04450_b200 import _native as nat
    nat.load().sc_trim_pool()
    torch.cuda.empty_cache()
    return out


def _extra(fn):
    """An extra full-size run reported beside the C2 line: a failure is
    reported in its key instead of losing the line."""
    try:
        return fn()
    except Exception as e:  # noqa: BLE001
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--ref-sample", type=int, default=8000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the public-API end-to-end timing (ncu runs)")
    ap.add_argument("--no-syn200", action="store_true", help="skip the extra Syn200 run (PAPER.md:536-550)")
    ap.add_argument("--no-c3", action="store_true",
                    help="skip the extra full-size C3 run (BASELINE.json configs[2] on this GPU) reported under 'c3'")
    ap.add_argument("--no-c5", action="store_true",
                    help="skip the extra full-size C5 k-means run (BASELINE.json configs[4]) reported under 'c5'")
    ap.add_argument("--c4", action="store_true",
                    help="also run full-size C4 (BASELINE.json configs[3], ~2-3 min) reported under 'c4'")
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
    x_host, y_planted = make_blobs(n, d, k, cs, seed=0)
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

    # timed steps: no per-kernel profiling events inside the timed region
    lib.sc_profile_enable(0)
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

    # one more step with the library's per-kernel CUDA events on (kernel
    # breakdown and the roofline's kernel time; not part of `value`)
    lib.sc_profile_reset()
    lib.sc_profile_enable(1)
    prof_steps = 1
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    device_step()
    e1.record()
    torch.cuda.synchronize()
    profiled_step_s = e0.elapsed_time(e1) / 1e3
    lib.sc_profile_enable(0)

    def prof(name):
        ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
        lib.sc_profile_query(name.encode(), nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
        return ms.value / prof_steps, cnt.value / prof_steps, work.value / prof_steps

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
    # (classes with algorithmic work only: knn_order is bookkeeping)
    dom = max((c for c in kstats if kstats[c][2] > 0), key=lambda c: kstats[c][0])
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
        "config": {"workload": f"{args.workload}: blobs N={n} d={d} kNN={knn} k={k} cs={cs} ({CONFIG_NOTE[args.workload]})",
                   "inputs": f"X resident in HBM ({x_host.nbytes / 1e6:.0f} MB; every stage's working set > L2)",
                   "parallelism":
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
        "step_stages_s": [{a: round(b, 3) for a, b in r.timings.items()} for r, _ in reports],
        "profiled_step_s": round(profiled_step_s, 4),
        "quality": {"ari_vs_planted": float(sc.adjusted_rand_index(rep.labeling.labels, y_planted)),
                    "max_eigen_residual": float(np.max(rep.eigen_residuals)),
                    "lambda_1": float(rep.eigenvalues[0]), "lambda_k": float(rep.eigenvalues[-1]),
                    "ncut": float(rep.ncut_value)},
        "eigen": {kk: v for kk, v in (dsc.last_info if sharded else __import__(
            "paper_1802_04450_b200.pipeline", fromlist=["x"]).last_info).get("eigen", {}).items() if kk != "history"},
    }
    clk = clocks.summary()
    line["clocks"] = clk
    if rank == 0 and world == 1 and not args.no_syn200:
        line["syn200"] = syn200_run(torch, sc, run_device)
    if rank == 0 and world == 1 and not args.no_c3 and args.workload != "c3":
        line["c3"] = _extra(lambda: c3_run(torch, sc, nat, run_device, lib))
    if rank == 0 and world == 1 and not args.no_c5:
        line["c5"] = _extra(lambda: c5_run(torch))
    if rank == 0 and world == 1 and args.c4:
        line["c4"] = _extra(lambda: c4_run(torch))
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # measured CPU baseline: the oracle port on the full C1 workload
        # (BASELINE.json configs[0], the reference's own CPU-runnable case),
        # and this engine on the same input, so the ratio is measured
        c1 = WORKLOADS["c1"]
        cpu_s, cpu_stages, cpu_labels, c1_y = oracle_run(*c1)
        xc1, _ = make_blobs(*[c1[i] for i in (0, 1, 3, 4)])
        n1, d1, knn1, k1, _ = c1
        cfg1 = sc.PipelineConfig(
            input=sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(float(np.sqrt(d1))), pattern="knn",
                                 points=xc1, knn=knn1),
            k_clusters=k1, eigen=sc.LanczosConfig(k=k1, seed=0), kmeans=sc.KmeansConfig(k=k1, seed=0),
            normalize_rows=True)
        sc.run(cfg1)
        g1 = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep1 = sc.run(cfg1)
            torch.cuda.synchronize()
            g1.append(time.perf_counter() - t0)
        cpu = host_cpu()
        line["cpu_baseline"] = {
            "value": cpu_s, "unit": "s", "cores": cpu["nproc"], "kind": "port", "cpu_model": cpu["model"],
            "sample": f"c1: oracle run_points on the full BASELINE configs[0] workload (blobs N={n1} d={d1} "
                      f"kNN={knn1} k={k1}), measured once; stages "
                      f"{{{', '.join(f'{a}: {b:.2f}' for a, b in cpu_stages.items())}}} s",
            "gpu_same_workload_s": float(np.median(g1)),
            "measured_ratio_c1": cpu_s / float(np.median(g1)),
            "ari_gpu_vs_cpu_labels": float(sc.adjusted_rand_index(rep1.labeling.labels, cpu_labels)),
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
