set -x
SPECLUST_TIMING_DEBUG=1 timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-c3 --no-e2e > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err
timeout 600 python tools/knn_modes.py c2 > gpurun_out/p_modes.json 2> gpurun_out/p_modes.err
python -c "
import json;d=json.loads(open('gpurun_out/p_bench.json').read().strip().splitlines()[-1])
for k in ['value','step_times_s','step_stages_s']: print(k, d.get(k))"; grep -E "knn_order|lanczos" gpurun_out/p_bench.err | awk '{print}' | sort | uniq -c | sort -rn | head -5; python - <<'PY'
import re
L=open('gpurun_out/p_bench.err').read().splitlines()
big=[l for l in L if re.search(r'([0-9.]+) ms', l) and float(re.search(r'([0-9.]+) ms', l).group(1))>40]
print('\n'.join(big[:40]))
PY
cat gpurun_out/p_modes.json; tail -3 gpurun_out/p_modes.err
