set -x
timeout 300 python tools/debug_lloyd.py > gpurun_out/r4_debug_lloyd.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reorth.py tests/test_gpu_shapes.py "tests/test_gpu_pipeline.py::test_pipeline_config1_full" -q -s > gpurun_out/r4_tests.log 2>&1
cat gpurun_out/r4_debug_lloyd.log; grep -E "passed|failed|FAILED|^E  |k=|ARI|subspace" gpurun_out/r4_tests.log | head -60
