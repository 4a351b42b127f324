set -x
timeout 300 python tools/block_micro.py > gpurun_out/d_block.json 2> gpurun_out/d_block.err
timeout 600 python tools/kmeans_c3.py > gpurun_out/d_km.json 2> gpurun_out/d_km.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:block_ -c 10 --csv python tools/block_micro.py > gpurun_out/d_block_ncu.csv 2>/dev/null
cat gpurun_out/d_block.json; tail -3 gpurun_out/d_block.err; cat gpurun_out/d_km.json; tail -3 gpurun_out/d_km.err
