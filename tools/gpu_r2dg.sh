timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/dg_tests.log 2>&1; tail -2 gpurun_out/dg_tests.log; grep -E "Error|assert " gpurun_out/dg_tests.log | head -5
timeout 1200 python bench.py > gpurun_out/dg_bench.json 2> gpurun_out/dg_bench.err; echo "bench rc=$?"
python - <<P
import json
d=json.loads(open('gpurun_out/dg_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['step_times_s'], d['stages_s'], d['kernels_ms_per_step']['reorth'], d['eigen'])
print('c3', d['c3']['seconds'], d['c3']['stages_s'], d['c3']['max_eigen_residual'], d['c3']['ari_vs_planted'], 'c5', d['c5']['seconds'], 'syn', d['syn200']['eigen_s'])
P
