timeout 900 python -m pytest tests/test_gpu_reorth.py tests/test_gpu_shapes.py tests/test_gpu_pipeline.py -q -x 2>&1 | tail -2
SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3 > gpurun_out/ca_c3.json 2> gpurun_out/ca_c3.err
grep "lanczos\] sweep" gpurun_out/ca_c3.err
python -c "import json;d=json.load(open('gpurun_out/ca_c3.json'));print(d['wall_s'],d['stages_s'],d['ari_vs_planted'],d['max_residual'],d['lambda'], d['eigen'])"
timeout 900 python tools/run_c4.py > gpurun_out/ca_c4.json 2> gpurun_out/ca_c4.err; tail -c 700 gpurun_out/ca_c4.json
