SPECLUST_SLOW_MS=15 timeout 300 python tools/step_var.py none 25 2> gpurun_out/bn.err | head -1
python - <<'PY'
import re
txt=open('gpurun_out/bn.err').read()
parts=re.split(r'=== step (\d+)\n',txt)
for i in range(1,len(parts),2):
    body=parts[i+1]
    m=re.search(r'=== end \d+ ([\d.]+)',body)
    wall=float(m.group(1)) if m else 0
    ls=[l for l in body.splitlines() if l.startswith('[slow]')]
    interesting=[l for l in ls if not re.match(r'\[slow\] (sc_knn_select_vals_f64|sc_eigensolve_csr_deflate|sc_eigensolve_csr) ',l)]
    print(parts[i], wall, ' | '.join(interesting)[:600])
PY
