d=gpurun_out
keys=()
while read -r v; do
  key=x$(printf '%s' "$v" | md5sum | cut -c1-7); keys+=($key)
  for alg in gradID FD ID Minv; do for dt in f64 f32; do
  RBD_PARTIAL_BUILD=1 RBD_TUNING="$v" RBD_BUILD_KEY=$key python tools/experiments/dump_outputs.py quad12 $alg $dt $d/o_${key}_${alg}_$dt.npz 8193 65541 2>&1 | tail -1
  done; done
done < tools/experiments/variants_q12trow2.txt
for k in ${keys[@]:1}; do for alg in gradID FD ID Minv; do for dt in f64 f32; do python tools/experiments/cmp_outputs.py $d/o_${keys[0]}_${alg}_$dt.npz $d/o_${k}_${alg}_$dt.npz | grep -c identical; done; done; done | sort | uniq -c
rm -f $d/o_*.npz
for alg in gradFD gradID FD ID Minv; do for dt in f64 f32; do
VARIANTS=tools/experiments/variants_q12trow2.txt bash tools/variants.sh time quad12 $alg $dt 1048576 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['alg'], d['dtype'], d['tuning'], d['N'], round(d['us'], 1))"
done; done
