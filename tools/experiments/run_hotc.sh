for r in chain7 quad12; do for i in 1 2; do
VARIANTS=tools/experiments/variants_hotc.txt bash tools/variants.sh time $r gradFD f64 1048576 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['robot'], d['tuning'], d['N'], round(d['us'], 1))"
done; done
