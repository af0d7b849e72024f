mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --print-kernel-base demangled \
    --log-file gpurun_out/launches_r15.csv \
    python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1
TAG=r15 SKIP_LAUNCHES=1 PROFILE_LIST="chain7 gradFD f64 1048576
chain7 gradFD f32 1048576" bash tools/gpu_profile.sh > /dev/null 2>&1
rm -f gpurun_out/*.ncu-rep
bash tools/gpu_state.sh > /dev/null 2>&1
tail -1 gpurun_out/pytest_gpu.log
