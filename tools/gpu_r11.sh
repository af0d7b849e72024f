mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --print-kernel-base demangled \
    --log-file gpurun_out/launches_r11.csv \
    python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1
TAG=r11 SKIP_LAUNCHES=1 PROFILE_LIST="chain7 gradFD f64 1048576
chain7 gradFD f32 1048576
quad12 gradFD f64 1048576" bash tools/gpu_profile.sh > /dev/null 2>&1
base=gpurun_out/prof_r11_humanoid30_gradFD_f64
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Knot_gradFD_f64_P0B -s 0 -c 1 -o $base -f python tools/profile_kernel.py --robot humanoid30 --alg gradFD --dtype f64 --n 65536 --launches 1 > $base.log 2>&1
ncu -i $base.ncu-rep --page raw --csv > $base.raw.csv 2>/dev/null
ncu -i $base.ncu-rep --page details --csv > $base.details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls gpurun_out | grep r11
