SPECLUST_TIMING_DEBUG=1 timeout 300 python tools/step_var.py sampler 14 2> gpurun_out/au_dbg.err | head -1
