set -x
timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_reorth.py "tests/test_gpu_kernels.py::test_lloyd_tensor_core_assignment_bit_identical" tests/test_gpu_pipeline.py -q -x > gpurun_out/c_tests.log 2>&1
timeout 2400 python tools/run_shape.py c3 > gpurun_out/c_c3.json 2> gpurun_out/c_c3.err
tail -5 gpurun_out/c_tests.log; cat gpurun_out/c_c3.json; tail -5 gpurun_out/c_c3.err
