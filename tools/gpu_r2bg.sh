timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/bg_tests.log 2>&1; tail -3 gpurun_out/bg_tests.log
SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3h > gpurun_out/bg_c3h.json 2> gpurun_out/bg_c3h.err
python -c "import json;d=json.load(open('gpurun_out/bg_c3h.json'));print(d['wall_s'],d['stages_s'],d['eigen'],d['ari_vs_planted'],d['max_residual'])"
SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3 > gpurun_out/bg_c3.json 2> gpurun_out/bg_c3.err
python -c "import json;d=json.load(open('gpurun_out/bg_c3.json'));print(d['wall_s'],d['stages_s'],d['eigen'],d['ari_vs_planted'],d['max_residual']); print({k:v['ms'] for k,v in d['kernels'].items()})"
