for dec in 5 6 7; do
SPECLUST_WDECADES=$dec timeout 900 python bench.py --no-c3 --no-c5 --no-syn200 --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/df_b.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/df_b.json').read().strip().splitlines()[-1]);print('dec=$dec c2', d['value'], [s['eigen'] for s in d['step_stages_s']], d['kernels_ms_per_step']['reorth'], d['eigen']['flushes'], d['eigen']['max_loss'], d['eigen']['mean_window'], d['quality']['max_eigen_residual'], d['eigen']['matvecs'])"
SPECLUST_WDECADES=$dec timeout 900 python tools/run_shape.py c3 > gpurun_out/df_c3.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/df_c3.json'));print('dec=$dec c3', d['wall_s'],d['stages_s']['eigen'],d['ari_vs_planted'],d['max_residual'], d['eigen'].get('max_loss'), d['eigen'].get('flushes'), d['eigen'].get('matvecs'))"
done
SPECLUST_WDECADES=7 timeout 900 python -m pytest tests/test_gpu_reorth.py tests/test_gpu_shapes.py -q -x 2>&1 | tail -2
