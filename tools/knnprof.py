import sys, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1802_04450_b200 as sc
from paper_1802_04450_b200.graph import knn_graph_device
from bench import make_blobs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
x, _ = make_blobs(n, 64, 100, 0.7)
xd = torch.from_numpy(x).cuda()
w, st = knn_graph_device(xd, 32, sc.SimilarityMeasure.exp_decay(8.0), return_stats=True)
torch.cuda.synchronize(); print(st)
