mkdir -p gpurun_out
i=0
for v in '{"trow_bk": 256}' '{"trow_bk": 256, "sync_every": 128}'; do
  i=$((i+1))
  key=x$(printf '%s' "$v" | md5sum | cut -c1-7)
  base=gpurun_out/prof_r2q_ls$i
  RBD_PARTIAL_BUILD=1 RBD_TUNING="$v" RBD_BUILD_KEY=$key timeout 900 ncu --set full --clock-control none --kernel-name-base demangled \
      -k regex:Knot_ -c 1 -o $base -f python tools/profile_kernel.py --robot chain7 --alg gradFD --dtype f64 --n 1048576 --launches 2 > $base.log 2>&1
  ncu -i $base.ncu-rep --page raw --csv > $base.raw.csv 2>/dev/null
  ncu -i $base.ncu-rep --page details --csv > $base.details.csv 2>/dev/null
  rm -f $base.ncu-rep
done
