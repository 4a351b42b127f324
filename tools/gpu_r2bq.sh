timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_distributed.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --sharded --workload c3h --steps 1 --warmup 1 --no-cpu-baseline --no-c3 --no-c5 --no-syn200 --no-e2e > gpurun_out/bq_sh.json 2> gpurun_out/bq_sh.err; tail -2 gpurun_out/bq_sh.err
python -c "
import json;d=json.loads(open('gpurun_out/bq_sh.json').read().strip().splitlines()[-1])
for k in ['value','stages_s','eigen','quality']: print(k, d.get(k))"
