# window CGS2 / flush reductions parallelised: GPU suite + C2 bench (no extras)
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/cl_tests.log 2>&1; tail -3 gpurun_out/cl_tests.log
timeout 900 python bench.py --no-c3 --no-c5 --no-syn200 --no-cpu-baseline > gpurun_out/cl_bench.json 2> gpurun_out/cl_bench.err
python - <<'P'
import json
d=json.loads(open('gpurun_out/cl_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['step_times_s'], d['stages_s'])
print(d['kernels_ms_per_step'])
print(d['eigen'])
P
