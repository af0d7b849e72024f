#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for spec in "chain7 gradFD f64" "chain7 gradFD f32" "quad12 gradFD f64" "humanoid30 gradFD f64" "humanoid30 gradFD f32"; do
  set -- $spec
  timeout 300 python tools/time_kernel.py --robot $1 --alg $2 --dtype $3 --n 1048576 128 256 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l); print(d['robot'], d['alg'], d['dtype'], d['N'], round(d['us'],1), '%.3g'%d['knots_per_s'])
    except Exception: print(l[:200])"
done
