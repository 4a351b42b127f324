timeout 600 python tools/spmv_sell_c2.py c2 placed band band32 > gpurun_out/dd_sp.json 2> gpurun_out/dd_sp.err; cat gpurun_out/dd_sp.json; tail -2 gpurun_out/dd_sp.err
SPECLUST_BAND_CHUNK=4096 timeout 600 python tools/spmv_sell_c2.py c2 band > gpurun_out/dd_sp2.json 2>> gpurun_out/dd_sp.err; cat gpurun_out/dd_sp2.json
