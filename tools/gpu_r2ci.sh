timeout 600 python tools/spmv_sell_c2.py c2 placed far1k far2k far4k far8k far16k > gpurun_out/ci_sp.json 2> gpurun_out/ci_sp.err; cat gpurun_out/ci_sp.json; tail -3 gpurun_out/ci_sp.err
