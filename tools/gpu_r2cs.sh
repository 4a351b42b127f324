SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3 > gpurun_out/cs_c3.json 2> gpurun_out/cs_c3.err
grep -i "kmeans++\|screen\|kpp\|k-means" gpurun_out/cs_c3.err | head -12
python -c "import json;d=json.load(open('gpurun_out/cs_c3.json'));print(d['wall_s'],d['stages_s'],d['ari_vs_planted'],d['max_residual'])"
