set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/f_tests.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:knn_cand_tc2 -c 1 -o gpurun_out/f_knn_src -f python tools/knn_once.py 200000 64 32 20 0.7 > gpurun_out/f_knn_ncu.log 2>&1
tail -5 gpurun_out/f_tests.log; python -c "
import json;d=json.loads(open('gpurun_out/f_bench.json').read().strip().splitlines()[-1]);print(d['value'],d.get('e2e'),d['stages_s'],d['kernels_ms_per_step'],d.get('eigen'),d.get('roofline'), d.get('cpu_baseline'), d.get('quality'))"; tail -3 gpurun_out/f_bench.err
