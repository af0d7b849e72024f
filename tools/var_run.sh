for spec in "chain7 f32" "quad12 f32" "quad12 f64"; do set -- $spec; VARIANTS=tools/variants_c7.txt bash tools/variants.sh time $1 gradFD $2 1048576 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l); print(d['robot'], d['dtype'], d['tuning'], round(d['us'],1), '%.3g'%d['knots_per_s'])
    except Exception: print(l[:200])"; done
