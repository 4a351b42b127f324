set -x
timeout 900 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_reorth.py -q -x > gpurun_out/n_acc.log 2>&1
timeout 900 python tools/diag_accept.py > gpurun_out/n_diag.txt 2>&1
timeout 600 python conformance/run_ref_suite.py --out gpurun_out > gpurun_out/n_conf.txt 2>&1
timeout 900 python tools/run_shape.py c3h > gpurun_out/n_c3h.json 2> gpurun_out/n_c3h.err
tail -15 gpurun_out/n_acc.log; cat gpurun_out/n_diag.txt | tail -12; tail -6 gpurun_out/n_conf.txt; python -c "
import json;d=json.load(open('gpurun_out/n_c3h.json')); print(d['wall_s'], d['stages_s'], d['eigen']); print({k:v['ms'] for k,v in d['kernels'].items()})"; tail -3 gpurun_out/n_c3h.err
