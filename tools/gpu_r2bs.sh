timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/bs_tests.log 2>&1; tail -3 gpurun_out/bs_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1500 python bench.py > gpurun_out/bs_bench.json 2> gpurun_out/bs_bench.err; tail -2 gpurun_out/bs_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bs_bench.json').read().strip().splitlines()[-1])
for k in ['value','e2e','stages_s','step_times_s','clocks','gpu_launches']: print(k, d.get(k))
print('roofline', {a: d['roofline'][a] for a in ['achieved','frac','kernel','ms_per_step']})
for k in ['c3','c5','syn200']:
    x=d.get(k,{}); print(k, {a:x.get(a) for a in ['seconds','stages_s','ari_vs_planted','s_per_iter','eigen_s','kmeans_s','error']})
print('cpu', {a: d['cpu_baseline'].get(a) for a in ['value','measured_ratio_c1','gpu_same_workload_s']})
PY
