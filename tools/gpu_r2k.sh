set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-c3 > gpurun_out/k_bench_ncu.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c3 > gpurun_out/k_bench.json 2> gpurun_out/k_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/k_bench.json').read().strip().splitlines()[-1])
for k in ['value','e2e','step_times_s','step_stages_s','syn200']: print(k, d.get(k))"; tail -3 gpurun_out/k_bench.err; wc -l gpurun_out/k_launches.csv
