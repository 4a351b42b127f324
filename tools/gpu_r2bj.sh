timeout 900 python -m pytest tests/test_gpu_pipeline.py -q -x -k "deflated" 2>&1 | tail -15
SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3h > gpurun_out/bj_c3h.json 2> gpurun_out/bj_c3h.err
python -c "import json;d=json.load(open('gpurun_out/bj_c3h.json'));print(d['wall_s'],d['stages_s'],d['eigen'],d['ari_vs_planted'],d['max_residual'])"
grep "lanczos\] restart\|sweep" gpurun_out/bj_c3h.err | tail -12
