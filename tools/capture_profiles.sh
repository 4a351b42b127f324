# Round profiling captures (1x B200): launch list of one C2 bench step and
# ncu --set full of the dominant kernels.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemv_t_partial -s 300 -c 1 \
  -o gpurun_out/ncu_gemv_t python tools/prof_lanczos.py > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemv_n_update -s 300 -c 1 \
  -o gpurun_out/ncu_gemv_n python tools/prof_lanczos.py > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spmv_local -s 5 -c 1 \
  -o gpurun_out/ncu_spmv python tools/prof_spmv.py perm > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"assign_tc_kernel<2" -s 3 -c 1 \
  -o gpurun_out/ncu_assign python tools/prof_lanczos.py > /dev/null 2>&1
ls -la gpurun_out
