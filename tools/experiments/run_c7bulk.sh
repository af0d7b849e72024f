set -x
d=gpurun_out
for v in '{}' '{"bulk_out": true}' '{"bulk_out": true, "l2_prefetch": 1}'; do
  key=x$(printf '%s' "$v" | md5sum | cut -c1-7)
  RBD_PARTIAL_BUILD=1 RBD_TUNING="$v" RBD_BUILD_KEY=$key python tools/experiments/dump_outputs.py chain7 gradFD f64 $d/o_$key.npz 1000 4096 65541
done
python tools/experiments/cmp_outputs.py $d/o_x99914b9.npz $d/o_x30858ad.npz
python tools/experiments/cmp_outputs.py $d/o_x99914b9.npz $d/o_x73c9c36.npz
rm -f $d/o_*.npz
VARIANTS=tools/experiments/variants_c7bulk.txt bash tools/variants.sh time chain7 gradFD f64 1048576 262144 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['tuning'], d['N'], round(d['us'], 1))"
