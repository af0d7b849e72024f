#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
bash tools/variants.sh time humanoid30 gradFD f64 262144 256 > gpurun_out/var3_h30_f64.jsonl 2>&1
bash tools/variants.sh time humanoid30 gradFD f32 262144 256 > gpurun_out/var3_h30_f32.jsonl 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/var3_*.jsonl')):
    for l in open(f):
        try: d=json.loads(l)
        except Exception: print(l[:300]); continue
        print(f[-20:], d['tuning'], d['N'], round(d['us'],1), '%.3g'%d['knots_per_s'], [ (p.get('registers'),p.get('spill_stores')) for p in d['ptxas']][:1])
PY
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; tail -2 gpurun_out/bench_r2.err
