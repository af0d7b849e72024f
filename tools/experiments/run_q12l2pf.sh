for r in 1 2; do
for dt in f64 f32; do for alg in gradFD FD; do
VARIANTS=tools/experiments/variants_q12l2pf.txt bash tools/variants.sh time quad12 $alg $dt 1048576 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['alg'], d['dtype'], d['tuning'], d['N'], round(d['us'], 1))"
done; done; done
