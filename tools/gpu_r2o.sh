set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/o_tests.log 2>&1
timeout 600 python conformance/run_ref_suite.py --out gpurun_out > gpurun_out/o_conf.txt 2>&1
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/o_bench.json 2> gpurun_out/o_bench.err
tail -5 gpurun_out/o_tests.log; tail -4 gpurun_out/o_conf.txt; python -c "
import json;d=json.loads(open('gpurun_out/o_bench.json').read().strip().splitlines()[-1])
for k in ['value','e2e','kernels_ms_per_step','roofline','step_times_s','clocks','cpu_baseline','syn200','c3']: print(k, d.get(k))"; tail -3 gpurun_out/o_bench.err
