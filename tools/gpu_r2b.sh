set -x
timeout 300 python -m pytest tests/test_gpu_io.py -q > gpurun_out/b_io.log 2>&1
timeout 900 python tools/run_shape.py c3h > gpurun_out/b_c3h.json 2> gpurun_out/b_c3h.err
timeout 1800 python tools/run_shape.py c3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
tail -3 gpurun_out/b_io.log; cat gpurun_out/b_c3h.json; tail -5 gpurun_out/b_c3h.err; cat gpurun_out/b_c3.json; tail -5 gpurun_out/b_c3.err
