mkdir -p gpurun_out
for n in 65536; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --print-kernel-base demangled --log-file gpurun_out/h30_parts.csv python tools/profile_kernel.py --robot humanoid30 --alg gradFD --dtype f64 --n $n --launches 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open('gpurun_out/h30_parts.csv')))
for i, r in enumerate(rows):
    if r and r[0] == "ID": h = r; st = i; break
k = h.index("Kernel Name"); v = h.index("Metric Value")
from collections import defaultdict
agg = defaultdict(float)
for r in rows[st+1:]: agg[r[k][:60]] += float(r[v].replace(',', ''))
for a, b in agg.items(): print(round(b/1e3, 1), "us", a)
PY
done
