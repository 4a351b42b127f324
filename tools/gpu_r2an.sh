set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "lloyd or kmeans or pairwise" > gpurun_out/ao_tests.log 2>&1
tail -3 gpurun_out/ao_tests.log
SPECLUST_ASSIGN_DEBUG=1 timeout 300 python tools/c5_once.py 10000000 6 2> gpurun_out/ao_c5.err; grep "tc kernel\|uncert" gpurun_out/ao_c5.err | head -30
timeout 900 python tools/run_c5.py > gpurun_out/ao_c5.json 2> gpurun_out/ao_c5r.err; cat gpurun_out/ao_c5.json; tail -3 gpurun_out/ao_c5r.err
