timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/cq_tests.log 2>&1; tail -3 gpurun_out/cq_tests.log
timeout 600 python -m pytest tests/test_gpu_reorth.py -q -s -k windowed_vs_full 2>&1 | grep -E "k=|passed|failed"
