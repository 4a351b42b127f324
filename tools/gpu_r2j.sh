set -x
SPECLUST_FLUSH_DEBUG=1 timeout 900 python tools/run_shape.py c3h > gpurun_out/j_c3h.json 2> gpurun_out/j_c3h.err
head -c 400 gpurun_out/j_c3h.json; grep -c flush gpurun_out/j_c3h.err
