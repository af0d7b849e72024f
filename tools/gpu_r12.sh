mkdir -p gpurun_out
base=gpurun_out/prof_r12_h30_P0B
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Knot_gradFD_f64_P0B -s 0 -c 1 -o $base -f python tools/profile_kernel.py --robot humanoid30 --alg gradFD --dtype f64 --n 32768 --launches 1 > $base.log 2>&1
ncu -i $base.ncu-rep --page source --csv --print-source sass > $base.sass.csv 2>/dev/null; gzip -f $base.sass.csv
rm -f $base.ncu-rep
