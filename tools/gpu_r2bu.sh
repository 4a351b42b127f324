nproc
for i in 1 2; do
STEPVAR_THREADS=1 timeout 300 python tools/step_var.py none 25 2> /dev/null | head -1
timeout 300 python tools/step_var.py none 25 2> /dev/null | head -1
done
