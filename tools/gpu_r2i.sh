set -x
SPECLUST_FLUSH_DEBUG=1 timeout 900 python tools/run_shape.py c3h > gpurun_out/i_c3h.json 2> gpurun_out/i_c3h.err
timeout 600 python tools/kmeans_c3.py > gpurun_out/i_km.json 2> gpurun_out/i_km.err
cat gpurun_out/i_c3h.json | head -c 600; grep -c flush gpurun_out/i_c3h.err; cat gpurun_out/i_km.json
