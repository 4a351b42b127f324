set -x
./tools/fp64_peak > gpurun_out/e_fp64.txt 2>&1
timeout 300 python tools/block_micro.py > gpurun_out/e_block.json 2> gpurun_out/e_block.err
timeout 600 python -m pytest tests/test_gpu_reorth.py tests/test_gpu_multirank.py -q -x > gpurun_out/e_tests.log 2>&1
timeout 600 python tools/kmeans_c3.py > gpurun_out/e_km.json 2> gpurun_out/e_km.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:knn_cand_tc2 -c 1 -o gpurun_out/e_knn_src -f python tools/knn_once.py 200000 64 32 20 0.7 > gpurun_out/e_knn_ncu.log 2>&1
cat gpurun_out/e_fp64.txt; cat gpurun_out/e_block.json; tail -3 gpurun_out/e_block.err; tail -15 gpurun_out/e_tests.log; cat gpurun_out/e_km.json; tail -3 gpurun_out/e_km.err; tail -3 gpurun_out/e_knn_ncu.log
