timeout 600 python tools/spmv_bound.py 2>&1 | tail -3
