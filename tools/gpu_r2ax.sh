for m in none sampler sampler5 none; do timeout 300 python tools/step_var.py $m 30 2> /dev/null | head -1; done
ps aux --sort=-%cpu | head -15
