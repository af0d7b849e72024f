mkdir -p gpurun_out
base=gpurun_out/prof_r5_humanoid30_gradFD_f64_P0
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:Knot_gradFD_f64_P0 -s 1 -c 1 -o $base -f \
      python tools/profile_kernel.py --robot humanoid30 --alg gradFD --dtype f64 --n 65536 --launches 2 > $base.log 2>&1
ncu -i $base.ncu-rep --page raw --csv > $base.raw.csv 2>/dev/null
ncu -i $base.ncu-rep --page details --csv > $base.details.csv 2>/dev/null
ncu -i $base.ncu-rep --page source --csv --print-source sass > $base.sass.csv 2>/dev/null; gzip -f $base.sass.csv
rm -f $base.ncu-rep
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --print-kernel-base demangled --log-file gpurun_out/h30_parts.csv python tools/profile_kernel.py --robot humanoid30 --alg gradFD --dtype f64 --n 262144 --launches 2 > /dev/null 2>&1
grep -o '"[^"]*Knot[^"]*","[^"]*","[^"]*","[^"]*"' gpurun_out/h30_parts.csv | head; grep "gpu__time" gpurun_out/h30_parts.csv | awk -F'","' '{print $5, $NF}' | head -20
