timeout 600 python tools/spmv_sell_c2.py c2 placed band band32 > gpurun_out/ck_sp.json 2> gpurun_out/ck_sp.err; cat gpurun_out/ck_sp.json; tail -3 gpurun_out/ck_sp.err
SPECLUST_BAND_CHUNK=2048 timeout 600 python tools/spmv_sell_c2.py c2 band > gpurun_out/ck_sp2.json 2>> gpurun_out/ck_sp.err; cat gpurun_out/ck_sp2.json
