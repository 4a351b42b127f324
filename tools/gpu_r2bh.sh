SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3h > gpurun_out/bh_c3h.json 2> gpurun_out/bh_c3h.err
grep "lanczos\] restart" gpurun_out/bh_c3h.err
