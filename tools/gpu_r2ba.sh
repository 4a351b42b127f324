for m in none sampler none; do timeout 300 python tools/step_var.py $m 30 2> /dev/null | grep -v "^{" | grep "^none\|^sampler\|cpu s"; done
