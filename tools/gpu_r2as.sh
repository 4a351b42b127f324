set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/as_tests.log 2>&1
tail -3 gpurun_out/as_tests.log
timeout 900 python tools/run_c5.py > gpurun_out/as_c5.json 2> gpurun_out/as_c5r.err; cat gpurun_out/as_c5.json; tail -3 gpurun_out/as_c5r.err
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/as_bench.json 2> gpurun_out/as_bench.err; tail -c 3000 gpurun_out/as_bench.json; tail -3 gpurun_out/as_bench.err
