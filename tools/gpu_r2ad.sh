set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py tests/test_gpu_shapes.py -q -x -k "knn or graph or pipeline or c3 or h3" > gpurun_out/ad_tests.log 2>&1
tail -3 gpurun_out/ad_tests.log
SPECLUST_KNN_TWOPASS=0 timeout 300 python tools/knn_pend.py c2 0 > gpurun_out/ad_one.json 2>&1; cat gpurun_out/ad_one.json
timeout 300 python tools/knn_pend.py c2 0 > gpurun_out/ad_two.json 2>&1; cat gpurun_out/ad_two.json
timeout 300 python tools/knn_pend.py c3h 0 > gpurun_out/ad_two_c3h.json 2>&1; cat gpurun_out/ad_two_c3h.json
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-c3 --no-syn200 --no-e2e > gpurun_out/ad_bench.json 2>gpurun_out/ad_bench.err; python -c "
import json;d=json.loads(open('gpurun_out/ad_bench.json').read().strip().splitlines()[-1])
for k in ['value','stages_s','kernels_ms_per_step','roofline']: print(k, d.get(k))"
