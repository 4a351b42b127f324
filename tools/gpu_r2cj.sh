timeout 600 python tools/spmv_sell_c2.py c2 placed band band32 band8 > gpurun_out/cj_sp.json 2> gpurun_out/cj_sp.err; cat gpurun_out/cj_sp.json; tail -3 gpurun_out/cj_sp.err
SPECLUST_BAND_CHUNK=4096 timeout 600 python tools/spmv_sell_c2.py c2 band band32 > gpurun_out/cj_sp2.json 2>> gpurun_out/cj_sp.err; cat gpurun_out/cj_sp2.json
