"""Locality-order experiment (host-side restatement of the kNN scan order in
csrc/sc_knn.cu: strided pivots refined by 4 Lloyd steps on a 32C subsample,
points bucketed by nearest pivot, buckets in pivot-tour order).  Measures,
for sampled query points, the fraction of their exact kNN that land within
+-W positions of the query in the order, for alternative pivot orders."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, d, knn, k, cs = bench.WORKLOADS[wl]
x, y = bench.make_blobs(n, d, k, cs)
x = (x - x.mean(0)).astype(np.float32)
C = min(1024, max(8, n // 1024))
piv = x[(np.arange(C) * n) // C].copy()
ns = min(n, 32 * C)
sub = x[(np.arange(ns) * n) // ns]


def sqd(a, b):
    return (a * a).sum(1)[:, None] + (b * b).sum(1)[None, :] - 2.0 * a @ b.T


for _ in range(4):
    lab = sqd(sub, piv).argmin(1)
    for c in range(C):
        m = lab == c
        if m.any():
            piv[c] = sub[m].mean(0)
D = np.maximum(sqd(piv, piv), 0)
t = time.time()
plab = np.empty(n, np.int64)
for s in range(0, n, 65536):
    plab[s:s + 65536] = sqd(x[s:s + 65536], piv).argmin(1)
print("assign", time.time() - t, file=sys.stderr)
rng = np.random.default_rng(1)
qs = rng.choice(n, 1500, replace=False)
nbr = np.empty((len(qs), knn), np.int64)
for s in range(0, len(qs), 250):
    dd = sqd(x[qs[s:s + 250]], x)
    dd[np.arange(len(dd)), qs[s:s + 250]] = np.inf
    nbr[s:s + 250] = np.argpartition(dd, knn, axis=1)[:, :knn]
print("knn", time.time() - t, file=sys.stderr)


def greedy_tour(D, start=0):
    C = len(D)
    used = np.zeros(C, bool)
    order = [start]
    used[start] = True
    cur = start
    for _ in range(C - 1):
        r = np.where(used, np.inf, D[cur])
        cur = int(r.argmin())
        used[cur] = True
        order.append(cur)
    return np.array(order)


def two_opt(order, D, passes=3):
    o = order.copy()
    C = len(o)
    for _ in range(passes):
        improved = False
        for i in range(1, C - 2):
            a, b = o[i - 1], o[i]
            c, dn = o[i + 1:C - 1], o[i + 2:C]
            delta = D[a, c] + D[b, dn] - D[a, b] - D[c, dn]
            j = int(np.argmin(delta))
            if delta[j] < -1e-9:
                jj = i + 1 + j
                o[i:jj + 1] = o[i:jj + 1][::-1].copy()
                improved = True
        if not improved:
            break
    return o


def two_level(D, G):
    # group pivots by k-medoids-like assignment to G greedy-farthest seeds, tour groups, tour inside
    C = len(D)
    seeds = [0]
    md = D[0].copy()
    for _ in range(G - 1):
        s = int(md.argmax())
        seeds.append(s)
        md = np.minimum(md, D[s])
    grp = D[:, seeds].argmin(1)
    # group distance = mean pivot distance
    GD = np.array([[D[np.ix_(grp == a, grp == b)].mean() for b in range(G)] for a in range(G)])
    gorder = two_opt(greedy_tour(GD), GD)
    out = []
    prev = None
    for g in gorder:
        mem = np.where(grp == g)[0]
        sub = D[np.ix_(mem, mem)]
        st = 0 if prev is None else int(D[prev, mem].argmin())
        o = two_opt(greedy_tour(sub, st), sub)
        out.extend(mem[o].tolist())
        prev = out[-1]
    return np.array(out)


def evaluate(name, porder):
    rank = np.empty(C, np.int64)
    rank[porder] = np.arange(C)
    key = rank[plab] * n + np.arange(n)
    pos = np.empty(n, np.int64)
    pos[np.argsort(key, kind="stable")] = np.arange(n)
    dist = np.abs(pos[nbr] - pos[qs][:, None])
    res = {W: float((dist <= W).mean()) for W in (1024, 8192, 65536)}
    tl = float(sum(D[porder[i], porder[i + 1]] for i in range(C - 1)))
    print(name, {"within": res, "tour_len": round(tl, 1)})


t0 = greedy_tour(D)
evaluate("greedy (current)", t0)
evaluate("greedy+2opt", two_opt(t0, D))
for G in (16, 32, 64, 128):
    evaluate(f"two-level G={G}", two_level(D, G))

# ceiling: pivots grouped by the majority planted blob of their bucket
maj = np.array([np.bincount(y[plab == c], minlength=k).argmax() if (plab == c).any() else 0 for c in range(C)])
evaluate("by planted blob", np.lexsort((np.arange(C), maj)))
# pure point order by planted blob (no pivots)
pos = np.empty(n, np.int64)
pos[np.argsort(y, kind="stable")] = np.arange(n)
dist = np.abs(pos[nbr] - pos[qs][:, None])
print("points by blob", {W: float((dist <= W).mean()) for W in (1024, 8192, 65536)})
print("same blob frac", float((y[nbr] == y[qs][:, None]).mean()))
