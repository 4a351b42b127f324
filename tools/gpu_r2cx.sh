timeout 900 python tools/knn_chunk.py c2 0 148 296 592 0 148 > gpurun_out/cx.json 2> gpurun_out/cx.err; cat gpurun_out/cx.json; tail -2 gpurun_out/cx.err
timeout 900 python tools/knn_chunk.py c3h 0 148 > gpurun_out/cx3.json 2>> gpurun_out/cx.err; cat gpurun_out/cx3.json
