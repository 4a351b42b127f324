"""Device Lloyd vs the oracle: pairwise distances by width, then which
iteration / quantity first differs."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_04450_b200 as sc
from oracle import speclust_oracle as orc
rng = np.random.default_rng(5)
for d in (16, 100, 128, 129, 130, 200, 256, 1000):
    v = rng.standard_normal((300, d)); c = rng.standard_normal((40, d))
    a = sc.pairwise_sq_dist(v, c); b = orc.pairwise_sq_dist(v, c)
    print(f"pairwise d={d}: equal {np.array_equal(a, b)} max rel {np.max(np.abs(a-b)/np.abs(b)):.2e}")
    nv = np.einsum("ij,ij->i", v, v)
    print(f"   sqnorm: einsum vs sum-of-squares loop equal? (host only)")
rng = np.random.default_rng(23)
for (n, d, k) in [(20_000, 100, 100), (20_000, 256, 1000)]:
    centers = rng.normal(0.0, 1.0, (k, d))
    v = centers[rng.integers(0, k, n)] + 0.3 * rng.standard_normal((n, d))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    init = v[rng.choice(n, k, replace=False)].copy()
    for it in (1, 2, 3):
        lab = sc.lloyd(v, init, sc.KmeansConfig(k=k, max_iters=it))
        l2, c2, sse, iters, hist = orc.lloyd(v, init, max_iters=it)
        dc = np.abs(lab.centroids - c2)
        print(f"n={n} d={d} k={k} iters={it}: labels equal {np.array_equal(lab.labels, l2)}, centroid max diff "
              f"{dc.max():.3e} ({int((dc > 0).sum())} entries), hist {lab.sse_history} vs {hist} diff "
              f"{np.abs(lab.sse_history - hist).max():.3e}")
        if (dc > 0).any():
            cl = int(np.argwhere(dc > 0)[0][0])
            prev = orc.lloyd(v, init, max_iters=it - 1)[0] if it > 1 else np.argmin(orc.pairwise_sq_dist(v, init), 1)
            mem = np.flatnonzero(prev == cl)
            s = np.zeros(d)
            for i in mem:
                s = s + v[i]
            print("   cluster", cl, "members", len(mem), "seq==oracle", np.array_equal(s / len(mem), c2[cl]),
                  "device==seq", np.array_equal(s / len(mem), lab.centroids[cl]))
            break
