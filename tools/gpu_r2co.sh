for v in 1e-6 1e-4 1e-2 0.1 0.5; do SPECLUST_WCANCEL=$v timeout 300 python tools/wcancel_probe.py 2>&1 | tail -1; done
