set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/a_gpu_tests.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
tail -n 40 gpurun_out/a_gpu_tests.log; python -c "
import json;d=json.loads(open('gpurun_out/a_bench.json').read().strip().splitlines()[-1]);print(d['value'],d.get('e2e'),d['stages_s'],d['kernels_ms_per_step'],d.get('eigen'),d.get('roofline'))"
