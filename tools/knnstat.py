import sys, time, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1802_04450_b200 as sc
from paper_1802_04450_b200.graph import knn_graph_device
from bench import make_blobs
x, _ = make_blobs(1_000_000, 64, 100, 0.7)
xd = torch.from_numpy(x).cuda()
m = sc.SimilarityMeasure.exp_decay(8.0)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    w, st = knn_graph_device(xd, 32, m, return_stats=True)
    torch.cuda.synchronize(); print("knn graph s", time.perf_counter() - t0, st, flush=True)
