#!/bin/bash
# ncu evidence: launch list of the bench + one full capture per kernel of interest.
# Reports are summarised on the box (raw/details CSV); only small .ncu-rep files
# come back (gpurun_out is capped at 64 MiB).
mkdir -p gpurun_out
TAG=${TAG:-r1}
if [ -z "$SKIP_LAUNCHES" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv --print-kernel-base demangled \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1
fi
while read -r robot alg dt n; do
  [ -z "$robot" ] && continue
  base=gpurun_out/prof_${TAG}_${robot}_${alg}_${dt}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:Knot_${alg}_${dt} -s 1 -c 1 -o $base -f \
      python tools/profile_kernel.py --robot $robot --alg $alg --dtype $dt --n $n --launches 2 > $base.log 2>&1
  ncu -i $base.ncu-rep --page raw --csv > $base.raw.csv 2>/dev/null
  ncu -i $base.ncu-rep --page details --csv > $base.details.csv 2>/dev/null
  ncu -i $base.ncu-rep --page source --csv --print-source sass > $base.sass.csv 2>/dev/null
  gzip -f $base.sass.csv
  sz=$(stat -c %s $base.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 12000000 ]; then rm -f $base.ncu-rep; fi
done <<< "${PROFILE_LIST:-chain7 gradFD f64 1048576}"
du -sh gpurun_out; ls -la gpurun_out
