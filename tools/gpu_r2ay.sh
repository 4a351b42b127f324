timeout 300 python tools/step_var.py none 20 2> /dev/null | grep -v "^{"
cat /proc/cpuinfo | grep "model name" | head -2; cat /sys/kernel/mm/transparent_hugepage/enabled; ls /sys/kernel/mm/damon/admin/kdamonds 2>/dev/null | head; cat /proc/sys/kernel/numa_balancing 2>/dev/null; free -g
