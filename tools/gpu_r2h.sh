set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_multirank.py tests/test_gpu_shapes.py -q -x > gpurun_out/h_tests.log 2>&1
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
tail -5 gpurun_out/h_tests.log; python -c "
import json;d=json.loads(open('gpurun_out/h_bench.json').read().strip().splitlines()[-1])
for k in ['value','e2e','stages_s','kernels_ms_per_step','roofline','step_times_s','profiled_step_s','cpu_baseline','c3']: print(k, d.get(k))"; tail -3 gpurun_out/h_bench.err
