"""C2 step-to-step variance probe: step times with and without the NVML
clock sampler, then (SPECLUST_TIMING_DEBUG set by the caller) per-phase logs
split per step by markers on fd 2."""
import os
import resource
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1802_04450_b200 as sc  # noqa: E402
from paper_1802_04450_b200 import pipeline as pl  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "sampler"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
n, d, knn, k, cs = bench.WORKLOADS["c2"]
x, _ = bench.make_blobs(n, d, k, cs)
xd = torch.from_numpy(x).cuda()
cfg = sc.PipelineConfig(
    input=sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(float(np.sqrt(d))), pattern="knn", points=xd, knn=knn),
    k_clusters=k, eigen=sc.LanczosConfig(k=k, seed=0), kmeans=sc.KmeansConfig(k=k, seed=0), normalize_rows=True)
if os.environ.get("STEPVAR_THREADS"):
    from threadpoolctl import threadpool_limits
    _tl = threadpool_limits(int(os.environ["STEPVAR_THREADS"]))
    torch.set_num_threads(int(os.environ["STEPVAR_THREADS"]))
    print("threads limited", file=sys.stderr)
sched = os.environ.get("STEPVAR_SCHED")
if sched:
    from cuda.bindings import runtime as rt
    flag = {"spin": rt.cudaDeviceScheduleSpin, "yield": rt.cudaDeviceScheduleYield,
            "block": rt.cudaDeviceScheduleBlockingSync}[sched]
    print("cudaSetDeviceFlags", sched, rt.cudaSetDeviceFlags(flag), rt.cudaGetDeviceFlags(), file=sys.stderr)
for _ in range(3):
    pl.run_device(cfg)
torch.cuda.synchronize()
times, stages, mem = [], [], []
ctx = bench.ClockSampler(0) if mode.startswith("sampler") else None
if mode == "sampler5":
    ctx.period = 0.5
if ctx:
    ctx.__enter__()
from paper_1802_04450_b200 import _native as nat  # noqa: E402
lib = nat.load()
classes = ["knn_order", "knn_tile", "knn_recheck", "knn_union", "spmv", "reorth", "ritz", "symeig", "embed",
           "kmeanspp", "kmeans_assign", "kmeans_update", "ncut"]
ksum, rus, steal = [], [], []
prof = os.environ.get("STEPVAR_PROF") is not None
for s in range(steps):
    os.write(2, f"=== step {s}\n".encode())
    r0 = resource.getrusage(resource.RUSAGE_SELF)
    st0 = [int(v) for v in open("/proc/stat").readline().split()[1:]]
    c0 = time.process_time()
    if prof:
        lib.sc_profile_reset()
        lib.sc_profile_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    rep, w = pl.run_device(cfg)
    e1.record()
    torch.cuda.synchronize()
    times.append(round(e0.elapsed_time(e1) / 1e3, 4))
    r1 = resource.getrusage(resource.RUSAGE_SELF)
    st1 = [int(v) for v in open("/proc/stat").readline().split()[1:]]
    steal.append([b - a for a, b in zip(st0, st1)])
    rus.append((round(time.process_time() - c0, 3), r1.ru_nivcsw - r0.ru_nivcsw, r1.ru_nvcsw - r0.ru_nvcsw,
                r1.ru_majflt - r0.ru_majflt, r1.ru_minflt - r0.ru_minflt))
    if prof:
        lib.sc_profile_enable(0)
        tot = 0.0
        for c in classes:
            ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
            lib.sc_profile_query(c.encode(), nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
            tot += ms.value
        ksum.append(round(tot, 1))
    stages.append({a: round(b, 3) for a, b in rep.timings.items()})
    os.write(2, f"=== end {s} {times[-1]} host {time.perf_counter() - t0:.4f}\n".encode())
    free, total = torch.cuda.mem_get_info()
    mem.append((round((total - free) / 1e9, 2), round(torch.cuda.memory_reserved() / 1e9, 2)))
if ctx:
    ctx.__exit__()
print(mode, times)
print("device used GB / torch reserved GB", mem)
print("kernel ms per step", ksum)
print("/proc/stat cpu deltas (user nice system idle iowait irq softirq steal)", [x[:8] for x in steal])
print("cpu s, invol csw, vol csw, majflt, minflt", rus)
for s in stages:
    print(s)
