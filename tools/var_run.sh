VARIANTS=tools/variants_c7.txt bash tools/variants.sh time chain7 gradFD f64 1048576 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l); print(d['dtype'], d['tuning'], round(d['us'],1), '%.3g'%d['knots_per_s'])
    except Exception: print(l[:200])"
