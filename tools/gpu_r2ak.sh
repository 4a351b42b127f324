set -x
SPECLUST_ASSIGN_DEBUG=1 timeout 300 python tools/run_c5.py 1000000 > gpurun_out/ak_c5_1m.json 2> gpurun_out/ak_c5_1m.err; cat gpurun_out/ak_c5_1m.json; grep assign_tc gpurun_out/ak_c5_1m.err | head -40
