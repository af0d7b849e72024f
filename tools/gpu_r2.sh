#!/bin/bash
# round-2 GPU pass: GPU tests, small-batch mappings, humanoid30 split variants, bench
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc $?"
tail -25 gpurun_out/pytest_$TAG.log
for r in chain7 quad12 humanoid30; do timeout 300 python tools/small_n.py $r gradFD,ID f64,f32 16,128,256,1024,4096; done > gpurun_out/small_n_$TAG.log 2>&1
grep -v '"ID"' gpurun_out/small_n_$TAG.log | head -40
python tools/time_kernel.py --robot humanoid30 --alg gradFD --dtype f64 --n 65536 262144 2>&1 | cut -c1-160
if [ -n "$SPLIT_VARIANTS" ]; then VARIANTS=$SPLIT_VARIANTS bash tools/variants.sh time humanoid30 gradFD f64 65536 262144 2>&1 | cut -c1-200; fi
t0=$(date +%s); timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc $? $(( $(date +%s) - t0 )) s"
tail -3 gpurun_out/bench_$TAG.err
