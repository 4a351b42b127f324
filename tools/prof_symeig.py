"""Profile helper: time the device symmetric eigensolver (sc_symeig_f64) on
a random m x m matrix; run under ncu for the per-kernel split."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1802_04450_b200 import _native as nat  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 200
k = m // 2
rng = np.random.default_rng(0)
t = rng.standard_normal((m, m))
t = t + t.T
lib = nat.load()
td = torch.from_numpy(np.asfortranarray(t).ravel(order="F")).cuda()
theta = torch.empty(m, dtype=torch.float64, device="cuda")
s = torch.empty((k, m), dtype=torch.float64, device="cuda")
for _ in range(3):
    nat.check(lib.sc_symeig_f64(m, k, nat.ptr(td), nat.ptr(theta), nat.ptr(s), nat.stream_handle()))
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    nat.check(lib.sc_symeig_f64(m, k, nat.ptr(td), nat.ptr(theta), nat.ptr(s), nat.stream_handle()))
torch.cuda.synchronize()
print(f"m={m}: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms per solve")
w = np.sort(np.linalg.eigvalsh(t))[::-1]
print("max |theta - lapack|", np.abs(theta.cpu().numpy() - w).max())
