timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x -k "deflated" 2>&1 | tail -2
timeout 1500 python bench.py --steps 5 --warmup 3 --c4 > gpurun_out/bl_bench.json 2> gpurun_out/bl_bench.err; tail -3 gpurun_out/bl_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bl_bench.json').read().strip().splitlines()[-1])
for k in ['value','e2e','stages_s','step_times_s','roofline','kernels_ms_per_step','eigen','quality']: print(k, d.get(k))
for k in ['c3','c4','c5','syn200']:
    x=d.get(k,{}); print(k, {a:x.get(a) for a in ['seconds','stages_s','eigen','ari_vs_planted','max_eigen_residual','s_per_iter','eigen_s','kmeans_s','assign_gemm','error']})
PY
