set -x
timeout 600 python -m pytest tests/test_gpu_symeig_dc.py tests/test_gpu_reorth.py -x -q -s > gpurun_out/r2_new_tests.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
tail -n 5 gpurun_out/r2_new_tests.log; tail -n 5 gpurun_out/r2_gpu_tests.log; head -c 2500 gpurun_out/r2_bench.json
