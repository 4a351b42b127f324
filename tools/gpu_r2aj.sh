set -x
timeout 300 python tools/run_c5.py 1000000 > gpurun_out/aj_c5_1m.json 2> gpurun_out/aj_c5_1m.err; cat gpurun_out/aj_c5_1m.json; tail -3 gpurun_out/aj_c5_1m.err
timeout 900 python tools/run_c5.py > gpurun_out/aj_c5.json 2> gpurun_out/aj_c5.err; cat gpurun_out/aj_c5.json; tail -3 gpurun_out/aj_c5.err
