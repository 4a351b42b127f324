set -x
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_distributed.py -q -x > gpurun_out/z_tests.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 2 --sharded --no-cpu-baseline --no-c3 --no-syn200 > gpurun_out/z_sharded.json 2> gpurun_out/z_sharded.err
tail -15 gpurun_out/z_tests.log; python -c "
import json;d=json.loads(open('gpurun_out/z_sharded.json').read().strip().splitlines()[-1])
for k in ['value','e2e','stages_s','kernels_ms_per_step','step_times_s','eigen','quality']: print(k, d.get(k))"; tail -3 gpurun_out/z_sharded.err
