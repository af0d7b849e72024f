d=gpurun_out
keys=()
while read -r v; do
  key=x$(printf '%s' "$v" | md5sum | cut -c1-7); keys+=($key)
  for alg in gradID Minv FD; do
  RBD_PARTIAL_BUILD=1 RBD_TUNING="$v" RBD_BUILD_KEY=$key python tools/experiments/dump_outputs.py chain7 $alg f64 $d/o_${key}_${alg}.npz 65541 2>&1 | tail -1
  done
done < tools/experiments/variants_c7trow_other.txt
for k in ${keys[@]:1}; do for alg in gradID Minv FD; do python tools/experiments/cmp_outputs.py $d/o_${keys[0]}_${alg}.npz $d/o_${k}_${alg}.npz; done; done | grep -c DIFFER
rm -f $d/o_*.npz
for alg in gradID Minv FD; do
VARIANTS=tools/experiments/variants_c7trow_other.txt bash tools/variants.sh time chain7 $alg f64 1048576 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['alg'], d['dtype'], d['tuning'], d['N'], round(d['us'], 1))"
done
