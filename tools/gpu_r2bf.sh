SPECLUST_FLUSH_DEBUG=1 SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3h > gpurun_out/bf_c3h.json 2> gpurun_out/bf_c3h.err; echo rc=$?
grep -c "ritz deciles" gpurun_out/bf_c3h.err; grep "ritz deciles" gpurun_out/bf_c3h.err | awk 'NR%8==1' | head -60
python -c "import json;d=json.load(open('gpurun_out/bf_c3h.json'));print(d['wall_s'],d['stages_s'],d['eigen'])"
