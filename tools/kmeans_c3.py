"""Time the k-means stage pieces at the C3 embedding shape (n x k unit rows,
k clusters): k-means++ seeding, Lloyd (tcgen05 assignment), per kernel class."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1802_04450_b200 import _native as nat  # noqa: E402
import paper_1802_04450_b200.kmeans  # noqa: E402,F401

km = sys.modules["paper_1802_04450_b200.kmeans"]

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
g = torch.Generator(device="cuda").manual_seed(0)
cent = torch.randn((k, k), generator=g, device="cuda", dtype=torch.float64)
y = torch.randint(0, k, (n,), generator=g, device="cuda")
v = cent[y] + 0.05 * torch.randn((n, k), generator=g, device="cuda", dtype=torch.float64)
v /= v.norm(dim=1, keepdim=True)
del cent
lib = nat.load()
out = {}
for rep in range(2):
    lib.sc_profile_reset()
    lib.sc_profile_enable(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows = km.kmeanspp_indices_device(v, k, 0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    init_c = v[torch.from_numpy(np.asarray(rows, dtype=np.int64)).cuda()].contiguous()
    labels, c, hist, it = km.lloyd_device(v, init_c, km.KmeansConfig(k=k, seed=0))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    kc = {}
    for name in ["kmeanspp", "kmeans_assign", "kmeans_update"]:
        ms, cnt, work = nat.C.c_double(), nat.C.c_int64(), nat.C.c_double()
        lib.sc_profile_query(name.encode(), nat.C.byref(ms), nat.C.byref(cnt), nat.C.byref(work))
        kc[name] = (round(ms.value, 2), cnt.value, work.value)
    out[rep] = {"kmeanspp_s": t1 - t0, "lloyd_s": t2 - t1, "iters": it, "kernels": kc}
print(json.dumps(out))
