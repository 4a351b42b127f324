set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/g_tests.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
timeout 900 python tools/run_shape.py c3h > gpurun_out/g_c3h.json 2> gpurun_out/g_c3h.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:knn_cand_tc2 -c 1 -o gpurun_out/g_knn_src -f python tools/knn_once.py 200000 64 32 20 0.7 > gpurun_out/g_knn_ncu.log 2>&1
tail -5 gpurun_out/g_tests.log; python -c "
import json;d=json.loads(open('gpurun_out/g_bench.json').read().strip().splitlines()[-1])
for k in ['value','e2e','stages_s','kernels_ms_per_step','eigen','roofline','quality','step_times_s','profiled_step_s']: print(k, d.get(k))"; tail -3 gpurun_out/g_bench.err; cat gpurun_out/g_c3h.json; tail -3 gpurun_out/g_c3h.err
