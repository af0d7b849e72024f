for dt in f32 f64; do VARIANTS=tools/variants_c7.txt bash tools/variants.sh time chain7 gradFD $dt 1048576 262144 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l); print(d['dtype'], d['N'], d['tuning'], round(d['us'],1), '%.3g'%d['knots_per_s'])
    except Exception: print(l[:200])"; done
