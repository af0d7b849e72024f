d=gpurun_out
for r in chain7; do
keys=()
while read -r v; do
  key=x$(printf '%s' "$v" | md5sum | cut -c1-7); keys+=($key)
  RBD_PARTIAL_BUILD=1 RBD_TUNING="$v" RBD_BUILD_KEY=$key python tools/experiments/dump_outputs.py $r gradFD f64 $d/o_${key}_$r.npz 65541 2>&1 | tail -1
done < tools/experiments/variants_sincos.txt
python tools/experiments/cmp_outputs.py $d/o_${keys[0]}_$r.npz $d/o_${keys[1]}_$r.npz
rm -f $d/o_*.npz
for i in 1 2; do
VARIANTS=tools/experiments/variants_sincos.txt bash tools/variants.sh time $r gradFD f64 1048576 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['robot'], d['alg'], d['dtype'], d['tuning'], d['N'], round(d['us'], 1))"
done; done
