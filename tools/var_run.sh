for dt in f64 f32; do VARIANTS=tools/variants_h30.txt bash tools/variants.sh time humanoid30 gradFD $dt 256 1024 2048 4096 8192 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l); print(d['robot'], d['alg'], d['dtype'], d['N'], d['tuning'], round(d['us'],2))
    except Exception: print(l[:200])"; done
