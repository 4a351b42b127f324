set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/l_tests.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c3 > gpurun_out/l_bench.json 2> gpurun_out/l_bench.err
timeout 600 python conformance/run_ref_suite.py --out gpurun_out > gpurun_out/l_conf.txt 2>&1
tail -5 gpurun_out/l_tests.log; python -c "
import json;d=json.loads(open('gpurun_out/l_bench.json').read().strip().splitlines()[-1])
for k in ['value','e2e','kernels_ms_per_step','roofline','step_times_s','syn200']: print(k, d.get(k))"; tail -3 gpurun_out/l_bench.err; tail -25 gpurun_out/l_conf.txt
