timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_shapes.py tests/test_gpu_pipeline.py -q -x > gpurun_out/ct_tests.log 2>&1; tail -2 gpurun_out/ct_tests.log; grep -E "Error|assert" gpurun_out/ct_tests.log | head -5
SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3 > gpurun_out/ct_c3.json 2> gpurun_out/ct_c3.err
grep -i "kmeans++" gpurun_out/ct_c3.err | head -5
python -c "import json;d=json.load(open('gpurun_out/ct_c3.json'));print(d['wall_s'],d['stages_s'],d['ari_vs_planted'],d['max_residual'])"
