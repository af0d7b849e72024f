d=gpurun_out
keys=()
while read -r v; do
  key=x$(printf '%s' "$v" | md5sum | cut -c1-7); keys+=($key)
  RBD_PARTIAL_BUILD=1 RBD_TUNING="$v" RBD_BUILD_KEY=$key python tools/experiments/dump_outputs.py quad12 gradFD f64 $d/o_$key.npz 8193 65541 2>&1 | tail -1
done < tools/experiments/variants_q12trow.txt
for k in ${keys[@]:1}; do python tools/experiments/cmp_outputs.py $d/o_${keys[0]}.npz $d/o_$k.npz; done
rm -f $d/o_*.npz
for r in 1 2; do
VARIANTS=tools/experiments/variants_q12trow.txt bash tools/variants.sh time quad12 gradFD f64 1048576 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['tuning'], d['N'], round(d['us'], 1), d['ptxas'][-1])"
done
