set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/v_tests.log 2>&1
SPECLUST_TIMING_DEBUG=1 timeout 1200 python tools/run_shape.py c3 > gpurun_out/v_c3.json 2> gpurun_out/v_c3.err
tail -4 gpurun_out/v_tests.log; grep -v "^\[lanczos\] sweep" gpurun_out/v_c3.err | tail -12; python -c "
import json;d=json.load(open('gpurun_out/v_c3.json')); print(d['wall_s'], d['stages_s']); print({k:v['ms'] for k,v in d['kernels'].items()})"
