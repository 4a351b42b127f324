set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "lloyd or kmeans or pairwise" > gpurun_out/al_tests.log 2>&1
tail -5 gpurun_out/al_tests.log
SPECLUST_ASSIGN_DEBUG=1 timeout 300 python tools/run_c5.py 1000000 > gpurun_out/al_c5_1m.json 2> gpurun_out/al_c5_1m.err; cat gpurun_out/al_c5_1m.json; grep assign_tc gpurun_out/al_c5_1m.err | head -24
timeout 900 python tools/run_c5.py > gpurun_out/al_c5.json 2> gpurun_out/al_c5.err; cat gpurun_out/al_c5.json; tail -3 gpurun_out/al_c5.err
