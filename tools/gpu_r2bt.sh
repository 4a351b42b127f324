timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -q -x -k "kmeans or kpp or pipeline" 2>&1 | tail -2
SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3 > gpurun_out/bt_c3.json 2> gpurun_out/bt_c3.err
python -c "import json;d=json.load(open('gpurun_out/bt_c3.json'));print(d['wall_s'],d['stages_s'],d['ari_vs_planted']); print({k:v['ms'] for k,v in d['kernels'].items() if 'kmeans' in k})"
timeout 600 python bench.py --steps 3 --warmup 3 --no-c3 --no-c5 --no-syn200 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['value'],d['step_times_s'],d['kernels_ms_per_step']['kmeanspp'],d['stages_s'])"
