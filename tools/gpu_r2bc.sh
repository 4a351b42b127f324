SPECLUST_TIMING_DEBUG=1 timeout 1500 python tools/run_c4.py > gpurun_out/bc_c4.json 2> gpurun_out/bc_c4.err; echo rc=$?
cat gpurun_out/bc_c4.json; grep -v "lanczos\] sweep" gpurun_out/bc_c4.err | tail -30; grep "lanczos\] sweep" gpurun_out/bc_c4.err | tail -5
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
