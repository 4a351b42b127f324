timeout 600 python tools/spmv_footprint.py c2 > gpurun_out/ch_fp.json 2> gpurun_out/ch_fp.err; cat gpurun_out/ch_fp.json; tail -3 gpurun_out/ch_fp.err
