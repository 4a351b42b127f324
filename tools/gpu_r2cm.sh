for v in A B C C; do
  cp tmpvar/lib$v.so paper_1802_04450_b200/libspeclust_b200.so
  echo "== $v"; timeout 600 python -m pytest tests/test_gpu_reorth.py -q -x -k "windowed_vs_full" -s 2>&1 | grep -E "k=|passed|failed|assert"
done
