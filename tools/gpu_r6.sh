mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --print-kernel-base demangled \
    --log-file gpurun_out/launches_r6.csv \
    python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1
TAG=r6 SKIP_LAUNCHES=1 PROFILE_LIST="chain7 gradFD f64 1048576
chain7 gradFD f32 1048576
quad12 gradFD f64 1048576" bash tools/gpu_profile.sh > /dev/null 2>&1
ls gpurun_out | grep r6
