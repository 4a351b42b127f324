set -x
SPECLUST_ASSIGN_DEBUG=1 timeout 300 python tools/c5_once.py 10000000 6 2> gpurun_out/am_c5.err; grep assign_tc gpurun_out/am_c5.err | head -30
timeout 600 ncu --set full --import-source on --clock-control none -k regex:assign_tc_kernel -c 1 -o gpurun_out/am_assign python tools/c5_once.py 1000000 1 > gpurun_out/am_ncu.log 2>&1; tail -3 gpurun_out/am_ncu.log
