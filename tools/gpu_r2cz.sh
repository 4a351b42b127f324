timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_shapes.py tests/test_gpu_pipeline.py -q -x > gpurun_out/cz_tests.log 2>&1; tail -2 gpurun_out/cz_tests.log; grep -E "Error|assert " gpurun_out/cz_tests.log | head -5
timeout 900 python tools/run_c5.py > gpurun_out/cz_c5.json 2> gpurun_out/cz_c5.err; python -c "
import json;d=json.load(open('gpurun_out/cz_c5.json'));print(d.get('seconds'), d.get('sse_last'), json.dumps(d.get('kernels'))[:400])"
timeout 900 python bench.py --no-c3 --no-c5 --no-syn200 --no-cpu-baseline --steps 7 > gpurun_out/cz_b.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/cz_b.json').read().strip().splitlines()[-1]);print(d['value'], d['step_times_s'], d['kernels_ms_per_step']['kmeans_update'], d['stages_s'])"
