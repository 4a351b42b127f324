nproc; uptime
timeout 300 python tools/step_var.py sampler 14 2> /dev/null | grep -v "^{"
STEPVAR_PROF=1 timeout 300 python tools/step_var.py sampler 14 2> /dev/null | grep -v "^{"
