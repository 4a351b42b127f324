set -x
SPECLUST_ASSIGN_DEBUG=1 timeout 300 python tools/c5_once.py 10000000 6 2> gpurun_out/ap_c5.err; grep "assign_tc\]" gpurun_out/ap_c5.err | grep -v rescanned | head -30
SPECLUST_ASSIGN_DEBUG=1 timeout 300 python tools/c5_once.py 1000000 6 2> gpurun_out/ap_c5m.err; grep "assign_tc\]" gpurun_out/ap_c5m.err | grep -v rescanned | head -30
