timeout 900 python -m pytest tests/test_gpu_pipeline.py -q -x -k "deflated" 2>&1 | tail -2
SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3 > gpurun_out/by_c3.json 2> gpurun_out/by_c3.err
python -c "import json;d=json.load(open('gpurun_out/by_c3.json'));print(d['wall_s'],d['stages_s'],d['ari_vs_planted'],d['max_residual']); print({k:v['ms'] for k,v in d['kernels'].items()})"
grep "lanczos\] sweep\|eigensolve" gpurun_out/by_c3.err | tail -5
