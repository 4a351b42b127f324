timeout 600 python tools/knn_margin.py c2 24 16 12 8 2>&1 | tail -1
