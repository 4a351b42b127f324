set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py tests/test_gpu_shapes.py -q -x -k "knn or graph or pipeline or c3 or h3" > gpurun_out/s_tests.log 2>&1
timeout 600 python tools/knn_modes.py c2 > gpurun_out/s_modes.json 2> gpurun_out/s_modes.err
tail -4 gpurun_out/s_tests.log; cat gpurun_out/s_modes.json; tail -2 gpurun_out/s_modes.err
