set -x
timeout 900 python tools/diag_accept.py > gpurun_out/m_diag.txt 2>&1
timeout 300 python tools/spmv_c2.py > gpurun_out/m_spmv.json 2> gpurun_out/m_spmv.err
cat gpurun_out/m_diag.txt | tail -40; cat gpurun_out/m_spmv.json; tail -3 gpurun_out/m_spmv.err
