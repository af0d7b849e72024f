bash tools/variants.sh time chain7 gradFD f64 1048576 128 > gpurun_out/var2_chain7_f64.jsonl 2>&1
bash tools/variants.sh time chain7 gradFD f32 1048576 128 > gpurun_out/var2_chain7_f32.jsonl 2>&1
bash tools/variants.sh time quad12 gradFD f64 1048576 128 > gpurun_out/var2_quad12_f64.jsonl 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/var2_*.jsonl')):
    for l in open(f):
        try: d=json.loads(l)
        except Exception: print(l[:200]); continue
        print(f[-20:], d['tuning'], d['N'], round(d['us'],1), '%.3g'%d['knots_per_s'], [ (p.get('registers'),p.get('spill_stores')) for p in d['ptxas']][:1])
PY
