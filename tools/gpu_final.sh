#!/bin/bash
# round-end evidence: GPU tests, bench line, ncu launch list of the bench
# command, one `ncu --set full` capture of the headline kernel, small-N table
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/pytest_$TAG.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc $?"; tail -2 gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --print-kernel-base demangled \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1; echo "launch list rc $?"
base=gpurun_out/prof_${TAG}_chain7_gradFD_f64
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Knot_ -c 1 -o $base -f \
    python tools/profile_kernel.py --robot chain7 --alg gradFD --dtype f64 --n 1048576 --launches 1 > /dev/null 2>&1; echo "ncu rc $?"
ncu -i $base.ncu-rep --page raw --csv > $base.raw.csv; ncu -i $base.ncu-rep --page details --csv > $base.details.csv
base=gpurun_out/prof_${TAG}_quad12_gradFD_f64
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Knot_ -c 1 -o $base -f \
    python tools/profile_kernel.py --robot quad12 --alg gradFD --dtype f64 --n 1048576 --launches 1 > /dev/null 2>&1; echo "ncu quad12 rc $?"
ncu -i $base.ncu-rep --page raw --csv > $base.raw.csv; ncu -i $base.ncu-rep --page details --csv > $base.details.csv
python tools/hbm_write_probe.py > gpurun_out/hbm_write_$TAG.json 2>&1; cat gpurun_out/hbm_write_$TAG.json
for r in chain7 quad12 humanoid30; do timeout 300 python tools/small_n.py $r gradFD,ID f64,f32 16,128,256,1024,4096; done > gpurun_out/small_n_$TAG.log 2>&1
ls -la gpurun_out | tail -12
