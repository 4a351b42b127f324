"""Host<->device round-trip latency over time: a tiny kernel + synchronize in
a loop for argv[1] seconds; prints the slow round trips (> 2 ms) with their
timestamps and a histogram (environment probe for step-time outliers)."""
import json
import sys
import time

import torch

dur = float(sys.argv[1]) if len(sys.argv) > 1 else 20.0
x = torch.zeros(1024, device="cuda")
torch.cuda.synchronize()
t_start = time.perf_counter()
slow = []
lat = []
while time.perf_counter() - t_start < dur:
    t0 = time.perf_counter()
    x.add_(1.0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    lat.append(dt)
    if dt > 2e-3:
        slow.append((round(t0 - t_start, 3), round(dt * 1e3, 2)))
import numpy as np  # noqa: E402
a = np.array(lat) * 1e6
print(json.dumps({"iters": len(lat), "p50_us": float(np.percentile(a, 50)), "p99_us": float(np.percentile(a, 99)),
                  "max_ms": float(a.max() / 1e3), "n_slow_gt2ms": len(slow), "slow": slow[:60]}))
