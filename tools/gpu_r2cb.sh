timeout 900 python -m pytest tests/test_gpu_reorth.py tests/test_gpu_shapes.py tests/test_gpu_pipeline.py -q -x 2>&1 | tail -2
