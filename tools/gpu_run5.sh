set -x
timeout 300 python tools/debug_lloyd.py > gpurun_out/r5_debug_lloyd.log 2>&1
timeout 900 python -m pytest tests/test_gpu_shapes.py "tests/test_gpu_kernels.py::test_lloyd_tensor_core_assignment_bit_identical" tests/test_gpu_kernels.py -q -x > gpurun_out/r5_tests.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r5_bench.json 2> gpurun_out/r5_bench.err
cat gpurun_out/r5_debug_lloyd.log | grep -v sqnorm; tail -n 15 gpurun_out/r5_tests.log; python -c "
import json;d=json.loads(open('gpurun_out/r5_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['stages_s'],d['kernels_ms_per_step'],d['eigen'])"
