timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "humanoid30" 2>&1 | tail -2
for alg in gradFD gradID; do for dt in f64 f32; do python tools/time_kernel.py --robot humanoid30 --alg $alg --dtype $dt --n 262144 | cut -c1-150; done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --print-kernel-base demangled --log-file gpurun_out/h30_split.csv python tools/profile_kernel.py --robot humanoid30 --alg gradFD --dtype f64 --n 65536 --launches 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open('gpurun_out/h30_split.csv')))
for i, r in enumerate(rows):
    if r and r[0] == "ID": h = r; st = i; break
k = h.index("Kernel Name"); v = h.index("Metric Value")
from collections import defaultdict
agg = defaultdict(float)
for r in rows[st+1:]: agg[r[k][:60]] += float(r[v].replace(',', ''))
for a, b in agg.items(): print(round(b/1e3, 1), "us", a)
PY
