d=gpurun_out
for r in quad12 tree7; do for alg in gradFD gradID Minv FD ID; do for dt in f64 f32; do
  RBD_PARTIAL_BUILD=1 RBD_BUILD_KEY=ff4c0f05 python tools/experiments/dump_outputs.py $r $alg $dt $d/o_old.npz 8193 65541 > /dev/null 2>&1
  RBD_PARTIAL_BUILD=1 RBD_BUILD_KEY=x99914b9 python tools/experiments/dump_outputs.py $r $alg $dt $d/o_new.npz 8193 65541 > /dev/null 2>&1
  echo "$r $alg $dt $(python tools/experiments/cmp_outputs.py $d/o_old.npz $d/o_new.npz | grep -c identical) identical"
done; done; done
rm -f $d/o_*.npz
for key in ff4c0f05 x99914b9; do for i in 1 2; do for alg in gradFD gradID FD; do for dt in f64 f32; do
  RBD_PARTIAL_BUILD=1 RBD_BUILD_KEY=$key timeout 300 python tools/time_kernel.py --robot quad12 --alg $alg --dtype $dt --n 1048576 | python -c "
import sys, json
d = json.loads(sys.stdin.readline()); print('$key', d['alg'], d['dtype'], round(d['us'], 1))"
done; done; done; done
