timeout 300 python tools/step_var.py sampler 12 2> /dev/null
timeout 300 python tools/step_var.py none 12 2> /dev/null
SPECLUST_TIMING_DEBUG=1 timeout 300 python tools/step_var.py sampler 12 2> gpurun_out/at_dbg.err | tail -20
