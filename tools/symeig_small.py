"""One small sc_symeig_f64 call (debugging aid)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_04450_b200 import _native as nat  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 9
k = max(1, m // 3)
rng = np.random.default_rng(m)
t = rng.standard_normal((m, m))
t = t + t.T
td = torch.from_numpy(t).cuda()
th = torch.empty(k, dtype=torch.float64, device="cuda")
s = torch.empty(m * k, dtype=torch.float64, device="cuda")
nat.check(nat.load().sc_symeig_f64(m, k, nat.ptr(td), nat.ptr(th), nat.ptr(s), nat.stream_handle()))
torch.cuda.synchronize()
print(m, th.cpu().numpy()[:3], np.sort(np.linalg.eigvalsh(t))[::-1][:3])
