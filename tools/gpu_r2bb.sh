timeout 900 python -m pytest tests/test_gpu_pipeline.py -q -x -k "basis or scaled or matrix" 2>&1 | tail -15
