set -x
SPECLUST_KNN_NOLIST=1 SPECLUST_KNN_TILE_ONLY=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:knn_cand_tc2 -c 1 -o gpurun_out/ag_nolist -f python tools/knn_once.py 200000 64 32 20 0.7 > gpurun_out/ag1.log 2>&1
SPECLUST_KNN_WAIT=19 SPECLUST_KNN_TILE_ONLY=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:knn_cand_tc2 -c 1 -o gpurun_out/ag_m19 -f python tools/knn_once.py 200000 64 32 20 0.7 > gpurun_out/ag2.log 2>&1
tail -2 gpurun_out/ag1.log gpurun_out/ag2.log
