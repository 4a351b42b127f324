SPECLUST_SELL_VARIANTS=4 timeout 600 python tools/spmv_sell_c2.py c2 placed pbal pbal32 p32x2 > gpurun_out/cf_sp.json 2> gpurun_out/cf_sp.err; cat gpurun_out/cf_sp.json; tail -3 gpurun_out/cf_sp.err
