SPECLUST_SELL_VARIANTS=0,4,8 timeout 600 python tools/spmv_sell_c2.py c2 placed local > gpurun_out/cd_sell.json 2> gpurun_out/cd_sell.err; cat gpurun_out/cd_sell.json; tail -3 gpurun_out/cd_sell.err
