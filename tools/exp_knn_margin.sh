#!/bin/bash
# kNN candidate margin sweep at C2 (tile time vs exact-fallback rows)
for M in 24 16 12 8; do
  echo "margin=$M"; SPECLUST_KNN_MARGIN=$M python tools/knn_time.py 1000000 64
done
