# re-entry check: full GPU suite + default bench at HEAD
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/cc_tests.log 2>&1; tail -3 gpurun_out/cc_tests.log
timeout 900 python bench.py > gpurun_out/cc_bench.json 2> gpurun_out/cc_bench.err; tail -c 600 gpurun_out/cc_bench.json
