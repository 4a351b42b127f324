timeout 1500 python tools/run_c4.py > gpurun_out/dc_c4.json 2> gpurun_out/dc_c4.err; echo "rc=$?"; tail -c 900 gpurun_out/dc_c4.json; tail -3 gpurun_out/dc_c4.err
