import sys, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1802_04450_b200 as sc
from paper_1802_04450_b200.graph import knn_graph_device
from oracle import speclust_oracle as orc
rng = np.random.default_rng(5)
for n, d, knn, scale in [(300, 3, 4, 1.0), (513, 17, 9, 0.3), (130, 64, 31, 3.0), (1000, 5, 1, 10.0), (1000, 5, 1, 1.0), (5000, 8, 4, 10.0)]:
    x = rng.standard_normal((n, d)) * scale
    sigma = float(np.sqrt(d))
    sel = orc.knn_selected(x, knn, sigma)
    w, st = knn_graph_device(x, knn, sc.SimilarityMeasure.exp_decay(sigma), return_stats=True)
    e = orc.knn_edges(x, knn, sigma)
    rp, col, _ = orc.csr_from_edges(n, e, orc.edge_weights(x, e, sigma))
    h = w.to_host()
    ok = np.array_equal(h.row_ptr, rp) and np.array_equal(h.col_idx, col)
    print(n, d, knn, scale, st, "OK" if ok else "MISMATCH", flush=True)
