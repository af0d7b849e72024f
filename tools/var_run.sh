VARIANTS=tools/variants_h30.txt bash tools/variants.sh time humanoid30 gradFD f64 262144 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l); print(d['dtype'], d['tuning'], round(d['us'],1), '%.3g'%d['knots_per_s'])
    except Exception: print(l[:200])"
