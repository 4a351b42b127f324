timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/bx_tests.log 2>&1; tail -2 gpurun_out/bx_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python bench.py > gpurun_out/bx_bench.json 2> gpurun_out/bx_bench.err; tail -2 gpurun_out/bx_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bx_ref.json 2> gpurun_out/bx_ref.err; tail -c 600 gpurun_out/bx_ref.json
timeout 900 python tools/run_c4.py > gpurun_out/bx_c4.json 2> gpurun_out/bx_c4.err; tail -c 800 gpurun_out/bx_c4.json
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bx_bench.json').read().strip().splitlines()[-1])
for k in ['value','e2e','stages_s','step_times_s','clocks','gpu_launches']: print(k, d.get(k))
print('roofline', {a: d['roofline'][a] for a in ['achieved','frac','kernel','ms_per_step']})
for k in ['c3','c5','syn200']:
    x=d.get(k,{}); print(k, {a:x.get(a) for a in ['seconds','stages_s','ari_vs_planted','s_per_iter','eigen_s','kmeans_s','error']})
PY
