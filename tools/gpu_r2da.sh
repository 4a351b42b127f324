for w in 16 32 16 32; do SPECLUST_WMAX0=$w SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3 > gpurun_out/da_c3.json 2> gpurun_out/da_c3.err
echo "wmax0=$w"; grep "lanczos\] sweep 0" gpurun_out/da_c3.err
python -c "import json;d=json.load(open('gpurun_out/da_c3.json'));print(d['wall_s'],d['stages_s']['eigen'],d['ari_vs_planted'],d['max_residual'], d['eigen'].get('max_loss'), d['eigen'].get('mean_window'))"; done
for w in 16 32; do SPECLUST_WMAX0=$w timeout 900 python bench.py --no-c3 --no-c5 --no-syn200 --no-cpu-baseline --steps 7 > gpurun_out/da_b.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/da_b.json').read().strip().splitlines()[-1]);print('c2 wmax0=$w', d['value'], [s['eigen'] for s in d['step_stages_s']], d['eigen'])"; done
