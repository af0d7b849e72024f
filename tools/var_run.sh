for spec in "humanoid30 gradFD f64 262144" "humanoid30 gradFD f32 262144" "quad12 gradFD f32 1048576" "quad12 gradID f64 1048576" "chain7 gradID f64 1048576" "chain7 FD f64 1048576" "chain7 Minv f64 1048576" "chain7 ID f64 1048576"; do set -- $spec; VARIANTS=tools/variants_h30.txt bash tools/variants.sh time $1 $2 $3 $4 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l); print(d['robot'], d['alg'], d['dtype'], d['tuning'], round(d['us'],1), '%.3g'%d['knots_per_s'])
    except Exception: print(l[:200])"; done
