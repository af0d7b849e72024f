for alg in gradFD gradID FD ID Minv; do for dt in f32 f64; do
VARIANTS=tools/experiments/variants_q12bk.txt bash tools/variants.sh time quad12 $alg $dt 1048576 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['alg'], d['dtype'], d['tuning'], round(d['us'], 1))"
done; done
