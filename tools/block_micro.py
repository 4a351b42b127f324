"""Bandwidth of the block Gram-Schmidt GEMMs (sc_block_tn_f64 / sc_block_nn_f64)
at Lanczos flush shapes."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1802_04450_b200 import _native as nat  # noqa: E402

lib = nat.load()
res = []
for n, nb, c in [(1_000_000, 150, 11), (1_000_000, 1500, 6), (1_000_000, 1500, 16), (4_000_000, 1500, 6),
                 (4_000_000, 1500, 32)]:
    ld = (n + 31) // 32 * 32
    B = torch.randn((nb + c) * ld, dtype=torch.float64, device="cuda")
    H = torch.empty(nb * c, dtype=torch.float64, device="cuda")
    V = B[nb * ld:]
    st = nat.stream_handle()
    for name in ("tn", "nn"):
        def run():
            if name == "tn":
                nat.check(lib.sc_block_tn_f64(n, ld, nb, nat.ptr(B), nat.ptr(V), c, nat.ptr(H), st))
            else:
                nat.check(lib.sc_block_nn_f64(n, ld, nb, nat.ptr(B), nat.ptr(H), c, nat.ptr(V), st))
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 5 / 1e3
        by = (nb + (c if name == "tn" else 2 * c)) * n * 8
        res.append({"op": name, "n": n, "nb": nb, "c": c, "ms": t * 1e3, "GBs": by / t / 1e9})
    del B, H, V
print(json.dumps(res))
