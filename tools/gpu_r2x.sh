# round-2 profile captures: C2 launch list (one pipeline run), a full ncu capture of the
# dominant kernel at C2 (DRAM traffic for roofline.traffic), smoke()
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-c3 --no-syn200 > gpurun_out/x_bench_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:knn_cand_tc2 -c 1 -o gpurun_out/x_knn_c2 -f python tools/knn_once.py 1000000 64 32 100 0.7 > gpurun_out/x_knn_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:spmv_placed -c 1 -o gpurun_out/x_spmv_c2 -f python tools/spmv_c2.py > gpurun_out/x_spmv_ncu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/x_smoke.log 2>&1
python tools/launch_summary.py gpurun_out/x_launches.csv | head -25; tail -2 gpurun_out/x_knn_ncu.log; tail -2 gpurun_out/x_spmv_ncu.log; tail -3 gpurun_out/x_smoke.log
