"""Full-size C5 (BASELINE.json configs[4]): Lloyd k-means on a 10M x 256
embedding with k = 10,000, a fixed 20 iterations from the reference's
``random_points`` init (SURVEY.md:594).  Prints one JSON line with the
seconds per iteration, the assignment GEMM's tensor-core rate and the
centroid update's bandwidth (profiled in a second, separate run)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
print(json.dumps(bench.c5_run(torch, n=n)))
