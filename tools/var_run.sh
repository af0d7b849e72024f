mkdir -p gpurun_out
VARIANTS=tools/variants_c7.txt bash tools/variants.sh time chain7 gradFD f64 1048576 > gpurun_out/var_c7_f64.jsonl 2>&1
VARIANTS=tools/variants_q12.txt bash tools/variants.sh time quad12 gradFD f64 1048576 > gpurun_out/var_q12_f64.jsonl 2>&1
for f in gpurun_out/var_*.jsonl; do python -c "
import json,sys
for l in open('$f'):
    try: d=json.loads(l); print(d['robot'],d['dtype'],d['tuning'],round(d['us'],1),'%.3g'%d['knots_per_s'], d['ptxas'])
    except Exception: print(l[:300])
"; done
