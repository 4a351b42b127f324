set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./tools/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_symeig_dc.py -x -q -s > gpurun_out/dc_tests.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err
tail -3 gpurun_out/dc_tests.log gpurun_out/gpu_tests.log; cat gpurun_out/fp64_peak.txt; cat gpurun_out/bench1.json | head -c 3000
