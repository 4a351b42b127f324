cat /sys/kernel/mm/damon/admin/kdamonds/*/state 2>/dev/null | head -3; ls /sys/kernel/mm/damon 2>/dev/null; cat /proc/sys/vm/swappiness; grep -i -E "thp|compact" /proc/vmstat | head -8
STEPVAR_MLOCK=1 timeout 300 python tools/step_var.py none 25 2> gpurun_out/bo.err | head -1; grep mlock gpurun_out/bo.err
timeout 300 python tools/step_var.py none 25 2> /dev/null | head -1
STEPVAR_MLOCK=1 timeout 300 python tools/step_var.py none 25 2> /dev/null | head -1
grep -i -E "thp|compact" /proc/vmstat | head -8
