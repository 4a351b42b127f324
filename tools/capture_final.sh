# End-of-round evidence (1x B200): the default bench line (no profiler), then
# the launch list of one C2 step and ncu --set full of the dominant kernels,
# each ncu pass after the plain run exited 0.  Outputs under gpurun_out/.
mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep
timeout 1200 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err || exit 1
tail -c 300 gpurun_out/fin_bench.json
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-c3 --no-c5 --no-syn200"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
  $B > gpurun_out/launches_bench.log 2>&1; echo "launch list rc=$?"
F="ncu --set full --import-source on --clock-control none"
timeout 900 $F -k regex:knn_cand_tc2 -c 1 -o gpurun_out/fin_knn_c2 $B > gpurun_out/fin_ncu_knn.log 2>&1; echo "knn rc=$?"
timeout 600 $F -k regex:spmv_placed -s 50 -c 1 -o gpurun_out/fin_spmv_c2 $B > gpurun_out/fin_ncu_spmv.log 2>&1; echo "spmv rc=$?"
timeout 600 $F -k regex:window_cgs2 -s 50 -c 1 -o gpurun_out/fin_wcgs2_c2 $B > gpurun_out/fin_ncu_wcgs2.log 2>&1; echo "wcgs2 rc=$?"
timeout 600 $F -k regex:kpp_update_panel -s 20 -c 1 -o gpurun_out/fin_kpp_c2 $B > gpurun_out/fin_ncu_kpp.log 2>&1; echo "kpp rc=$?"
timeout 600 $F -k regex:block_reduce -s 20 -c 1 -o gpurun_out/fin_breduce_c2 $B > gpurun_out/fin_ncu_breduce.log 2>&1; echo "breduce rc=$?"
ls -la gpurun_out/*.ncu-rep
