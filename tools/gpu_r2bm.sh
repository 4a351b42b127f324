timeout 120 python tools/sync_latency.py 30
