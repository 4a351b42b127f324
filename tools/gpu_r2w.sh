set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/w_tests.log 2>&1
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/w_bench.json 2> gpurun_out/w_bench.err
tail -4 gpurun_out/w_tests.log; python -c "
import json;d=json.loads(open('gpurun_out/w_bench.json').read().strip().splitlines()[-1])
for k in ['value','e2e','kernels_ms_per_step','roofline','step_times_s','clocks','syn200','c3']: print(k, d.get(k))"; tail -3 gpurun_out/w_bench.err
