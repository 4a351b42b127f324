# step variance vs the in-process NVML clock sampler period
for per in 0.1 1000 0.1 1000 0.1 1000; do SPECLUST_CLOCK_PERIOD=$per timeout 900 python bench.py --no-c3 --no-c5 --no-syn200 --no-cpu-baseline --steps 9 > gpurun_out/cw_b.json 2>/dev/null
python - <<P
import json
d=json.loads(open('gpurun_out/cw_b.json').read().strip().splitlines()[-1])
print("period=$per", round(d['value'],4), round(d['e2e']['value'],4), d['step_times_s'], d['clocks'].get('samples'))
P
done
