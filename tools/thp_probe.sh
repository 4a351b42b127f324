for f in enabled defrag khugepaged/defrag; do echo "$f: $(cat /sys/kernel/mm/transparent_hugepage/$f 2>&1)"; done
cat /proc/sys/vm/compaction_proactiveness 2>&1; nproc; free -g | head -2
grep -i "damon" /proc/modules 2>/dev/null | head -2; ls /sys/kernel/mm/damon 2>&1 | head -3
