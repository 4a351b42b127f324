SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c3 > gpurun_out/bz_c3.json 2> gpurun_out/bz_c3.err
grep "lanczos\] sweep" gpurun_out/bz_c3.err
SPECLUST_TIMING_DEBUG=1 timeout 900 python tools/run_shape.py c2 > gpurun_out/bz_c2.json 2> gpurun_out/bz_c2.err
grep "lanczos\] sweep" gpurun_out/bz_c2.err
