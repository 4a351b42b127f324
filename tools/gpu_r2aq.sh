set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -q -x -k "lloyd or kmeans or pairwise or pipeline" > gpurun_out/ar_tests.log 2>&1
tail -3 gpurun_out/ar_tests.log
SPECLUST_ASSIGN_DEBUG=1 timeout 300 python tools/c5_once.py 10000000 6 2> gpurun_out/ar_c5.err; grep "assign_tc\]" gpurun_out/ar_c5.err | grep -v rescanned | head -30
SPECLUST_FINALIZE=panel SPECLUST_ASSIGN_DEBUG=1 timeout 300 python tools/c5_once.py 10000000 3 2> gpurun_out/ar_c5p.err; grep "assign_tc\]" gpurun_out/ar_c5p.err | grep -v rescanned | head -30
SPECLUST_ASSIGN_DEBUG=1 timeout 300 python tools/c5_once.py 1000000 6 2> gpurun_out/ar_c5m.err; grep "assign_tc\]" gpurun_out/ar_c5m.err | grep -v rescanned | head -30
timeout 900 python tools/run_c5.py > gpurun_out/ar_c5.json 2> gpurun_out/ar_c5r.err; cat gpurun_out/ar_c5.json; tail -3 gpurun_out/ar_c5r.err
