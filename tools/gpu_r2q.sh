set -x
timeout 300 python tools/spmv_c2.py > gpurun_out/q_spmv.json 2> gpurun_out/q_spmv.err
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,dram__bytes_read.sum --clock-control none -k regex:spmv_ -c 12 --csv python tools/spmv_c2.py > gpurun_out/q_spmv_ncu.csv 2>/dev/null
SPECLUST_SPMV_KERNEL=placed timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k spmv > gpurun_out/q_tests.log 2>&1
cat gpurun_out/q_spmv.json; tail -3 gpurun_out/q_spmv.err; tail -3 gpurun_out/q_tests.log; grep -E "spmv_(local|placed|pipe)" gpurun_out/q_spmv_ncu.csv | awk -F'","' '{print $5" | "$(NF-2)" | "$NF}' | cut -c1-150 | head -30
