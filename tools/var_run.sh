for i in 1 2; do VARIANTS=tools/variants_c7.txt bash tools/variants.sh time chain7 gradFD f64 16 128 256 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l); print(d['N'], d['tuning'], round(d['us'],2))
    except Exception: print(l[:200])"; done
