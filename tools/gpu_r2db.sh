# end of round: GPU suite, smoke(), default bench line
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/db_tests.log 2>&1; tail -2 gpurun_out/db_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/db_bench.json 2> gpurun_out/db_bench.err; echo "bench rc=$?"
python - <<P
import json
d=json.loads(open('gpurun_out/db_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['step_times_s'], d['stages_s'])
print('c3', d['c3']['seconds'], d['c3']['stages_s'], 'c5', d['c5']['seconds'], 'syn', d['syn200']['eigen_s'], d['syn200']['kmeans_s'])
print(d['roofline']['frac'], d['spmv_frac_hbm'], d['clocks'], d['gpu_launches'])
P
