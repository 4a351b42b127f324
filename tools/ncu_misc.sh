#!/bin/bash
# ncu --set full of one launch each of the CSR permutation, k-means++ update and
# certified-assignment finalize kernels at C2 shape
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:perm_row_fill -c 1 \
  -o gpurun_out/ncu_perm -f python tools/prof_spmv.py perm > gpurun_out/ncu_perm.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kpp_update -s 50 -c 1 \
  -o gpurun_out/ncu_kpp -f python tools/prof_lanczos.py > gpurun_out/ncu_kpp.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:as_finalize -s 5 -c 1 \
  -o gpurun_out/ncu_fin -f python tools/prof_lanczos.py > gpurun_out/ncu_fin.log 2>&1
