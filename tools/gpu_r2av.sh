timeout 300 python tools/step_var.py sampler 14 2> /dev/null | head -2
