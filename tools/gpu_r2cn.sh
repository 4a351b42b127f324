for v in H C; do
  cp tmpvar/lib$v.so paper_1802_04450_b200/libspeclust_b200.so
  echo "== $v"; SPECLUST_FLUSH_DEBUG=1 timeout 600 python -m pytest tests/test_gpu_reorth.py -q -x -k "windowed_vs_full and 100" -s > gpurun_out/cn_$v.log 2>&1; grep -E "k=|passed|failed" gpurun_out/cn_$v.log
done
