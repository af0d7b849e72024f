d=gpurun_out
keys=()
while read -r v; do
  key=x$(printf '%s' "$v" | md5sum | cut -c1-7); keys+=($key)
  for alg in gradFD gradID Minv; do
  RBD_PARTIAL_BUILD=1 RBD_TUNING="$v" RBD_BUILD_KEY=$key python tools/experiments/dump_outputs.py quad12 $alg f64 $d/o_${key}_${alg}.npz 65541 2>&1 | tail -1
  done
done < tools/experiments/variants_q12ctas.txt
for k in ${keys[@]:1}; do for alg in gradFD gradID Minv; do python tools/experiments/cmp_outputs.py $d/o_${keys[0]}_${alg}.npz $d/o_${k}_${alg}.npz; done; done | grep -c DIFFER
rm -f $d/o_*.npz
for r in 1 2; do for alg in gradFD gradID Minv; do
VARIANTS=tools/experiments/variants_q12ctas.txt bash tools/variants.sh time quad12 $alg f64 1048576 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['alg'], d['dtype'], d['tuning'], d['N'], round(d['us'], 1))"
done; done
