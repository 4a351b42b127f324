"""Full-size C4 (BASELINE.json configs[3]) on one GPU: bench.c4_run as one JSON line."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

print(json.dumps(bench.c4_run(torch)))
