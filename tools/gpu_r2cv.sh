bash tools/thp_probe.sh
for t in 1 0 1 0; do SPECLUST_NO_THP=$t timeout 900 python bench.py --no-c3 --no-c5 --no-syn200 --no-cpu-baseline --steps 7 > gpurun_out/cv_b$t.json 2>/dev/null
python - <<P
import json
d=json.loads(open('gpurun_out/cv_b$t.json').read().strip().splitlines()[-1])
print("no_thp=$t", d['value'], d['e2e']['value'], d['step_times_s'])
P
done
