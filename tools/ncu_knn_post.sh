#!/bin/bash
# ncu --set full of the kNN post-candidate kernels at C2 shape (args: n d)
mkdir -p gpurun_out
for k in ${KERNELS:-knn_recheck_kernel row_fill_vals_kernel}; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/ncu_$k -f python tools/knn_time.py ${1:-1000000} ${2:-64} > gpurun_out/ncu_$k.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/knn_launches.csv python tools/knn_time.py ${1:-1000000} ${2:-64} > /dev/null 2>&1
