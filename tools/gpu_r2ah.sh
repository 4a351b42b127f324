set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py tests/test_gpu_shapes.py -q -x -k "knn or graph or pipeline or c3 or h3" > gpurun_out/ah_tests.log 2>&1
tail -3 gpurun_out/ah_tests.log
bash tools/gpu_r2aa.sh > /dev/null 2>&1; cat gpurun_out/aa_modes.txt
timeout 300 python tools/knn_pend.py c2 0 > gpurun_out/ah_c2.json 2>&1; cat gpurun_out/ah_c2.json
timeout 300 python tools/knn_pend.py c3h 0 > gpurun_out/ah_c3h.json 2>&1; cat gpurun_out/ah_c3h.json
