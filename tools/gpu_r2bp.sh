set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bp_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-c3 --no-c5 --no-syn200 > gpurun_out/bp_bench_ncu.log 2>&1
tail -2 gpurun_out/bp_bench_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:assign_tc_kernel -s 3 -c 1 -o gpurun_out/bp_assign python tools/c5_once.py 1000000 6 > gpurun_out/bp_ncu_assign.log 2>&1
tail -2 gpurun_out/bp_ncu_assign.log
