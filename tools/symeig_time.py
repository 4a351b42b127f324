"""Time the device projected eigensolver (sc_symeig_f64) on a Lanczos-like
m x m matrix (clustered top eigenvalues) and check it against numpy.
python tools/symeig_time.py [m ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_04450_b200 import _native as nat  # noqa: E402

lib = nat.load()
for m in [int(a) for a in sys.argv[1:]] or [200, 2000]:
    rng = np.random.default_rng(m)
    q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    lam = np.concatenate([1.0 - 0.002 * rng.random(m // 2), rng.random(m - m // 2) * 0.9])
    t = (q * lam) @ q.T
    t = (t + t.T) / 2
    k = m // 2
    td = torch.from_numpy(np.ascontiguousarray(t)).cuda()
    th = torch.empty(k, dtype=torch.float64, device="cuda")
    s = torch.empty(m * k, dtype=torch.float64, device="cuda")
    st = nat.stream_handle()
    nat.check(lib.sc_symeig_f64(m, k, nat.ptr(td), nat.ptr(th), nat.ptr(s), st))
    torch.cuda.synchronize()
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        nat.check(lib.sc_symeig_f64(m, k, nat.ptr(td), nat.ptr(th), nat.ptr(s), st))
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    w = np.sort(np.linalg.eigvalsh(t))[::-1][:k]
    got = th.cpu().numpy()
    sv = s.cpu().numpy().reshape(k, m).T
    res = np.abs(t @ sv - sv * got).max()
    print(f"m={m} k={k}: {dt * 1e3:.1f} ms/call  max|dtheta| {np.abs(got - w).max():.2e}  max residual {res:.2e}")
