set -x
timeout 900 python -m pytest tests/test_gpu_reorth.py tests/test_gpu_shapes.py "tests/test_gpu_kernels.py::test_sbm_long_rows" "tests/test_gpu_kernels.py::test_lloyd_tensor_core_assignment_bit_identical" -q -s > gpurun_out/r3_new_tests.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3_gpu_tests.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3_bench.json 2> gpurun_out/r3_bench.err
tail -n 30 gpurun_out/r3_new_tests.log; tail -n 5 gpurun_out/r3_gpu_tests.log; head -c 2500 gpurun_out/r3_bench.json
