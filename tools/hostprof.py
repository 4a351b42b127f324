import sys, time, cProfile, pstats, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1802_04450_b200 as sc
from paper_1802_04450_b200.pipeline import run_device
from bench import make_blobs
x, _ = make_blobs(1_000_000, 64, 100, 0.7)
xd = torch.from_numpy(x).cuda()
cfg = sc.PipelineConfig(input=sc.PointsInput(measure=sc.SimilarityMeasure.exp_decay(8.0), pattern="knn", points=xd, knn=32),
                        k_clusters=100, eigen=sc.LanczosConfig(k=100, seed=0), kmeans=sc.KmeansConfig(k=100, seed=0), normalize_rows=True)
for i in range(3):
    t0 = time.perf_counter(); rep, w = run_device(cfg); torch.cuda.synchronize()
    print(i, round(time.perf_counter() - t0, 3), {k: round(v, 3) for k, v in rep.timings.items()}, flush=True)
pr = cProfile.Profile(); pr.enable()
rep, w = run_device(cfg); torch.cuda.synchronize()
pr.disable()
print({k: round(v, 3) for k, v in rep.timings.items()})
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
