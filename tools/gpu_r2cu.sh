timeout 600 python -m pytest tests/test_gpu_lookahead.py -q -x > gpurun_out/cu_la.log 2>&1; tail -3 gpurun_out/cu_la.log; grep -E "Error|assert " gpurun_out/cu_la.log | head -5
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/cu_tests.log 2>&1; tail -2 gpurun_out/cu_tests.log
for la in 1 0 1 0; do SPECLUST_LOOKAHEAD=$la timeout 900 python bench.py --no-c3 --no-c5 --no-syn200 --no-cpu-baseline --steps 7 > gpurun_out/cu_b$la.json 2>/dev/null
python - <<P
import json
d=json.loads(open('gpurun_out/cu_b$la.json').read().strip().splitlines()[-1])
print("lookahead=$la", d['value'], d['e2e']['value'], d['step_times_s'], [s['eigen'] for s in d['step_stages_s']])
P
done
SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3 > gpurun_out/cu_c3.json 2> gpurun_out/cu_c3.err
grep "lanczos\] sweep" gpurun_out/cu_c3.err
python -c "import json;d=json.load(open('gpurun_out/cu_c3.json'));print(d['wall_s'],d['stages_s'],d['ari_vs_planted'],d['max_residual'])"
