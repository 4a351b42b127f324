"""Windowed Lanczos on the C4-shape SBM golden operator (the reorth test's
case) and on C2: max flush loss, whole-basis passes and solve time as the
window-cancellation threshold (SPECLUST_WCANCEL) varies."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1802_04450_b200 as sc  # noqa: E402
from paper_1802_04450_b200.eigen import eigensolve_device  # noqa: E402

g = np.load("tests/golden/shape_c4s.npz")
n = len(g["row_ptr"]) - 1
w = sc.CsrMatrix(n, n, g["row_ptr"].astype(np.int64), g["col"].astype(np.int64), np.ones(len(g["col"])))
a = sc.sym_scale(w, sc.degrees(w)).device()
os.environ["SPECLUST_REORTH"] = "window"
out = {}
for k in (100, 1000):
    torch.cuda.synchronize()
    t = time.perf_counter()
    vals, vecs, res, st = eigensolve_device(a, sc.LanczosConfig(k=k, seed=0))
    torch.cuda.synchronize()
    U = vecs.cpu().numpy()
    out[f"sbm_k{k}"] = {"max_loss": st["max_loss"], "second_passes": st["second_passes"], "flushes": st["flushes"],
                        "matvecs": st["matvecs"], "s": time.perf_counter() - t, "max_res": float(np.max(res)),
                        "orth": float(np.abs(U.T @ U - np.eye(k)).max())}
print(json.dumps({"wcancel": os.environ.get("SPECLUST_WCANCEL", "default"), **out}))
