STEPVAR_SCHED=spin timeout 300 python tools/step_var.py none 30 2> gpurun_out/az_spin.err | grep -v "^{" | grep "none\|cpu s"; grep cudaSet gpurun_out/az_spin.err
timeout 300 python tools/step_var.py none 30 2> /dev/null | grep -v "^{" | grep "none\|cpu s"
STEPVAR_SCHED=spin timeout 300 python tools/step_var.py none 30 2> /dev/null | grep -v "^{" | grep "none"
STEPVAR_SCHED=block timeout 300 python tools/step_var.py none 12 2> /dev/null | grep -v "^{" | grep "none"
