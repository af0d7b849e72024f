#!/bin/bash
# ncu --set full captures: one line per capture "robot alg dtype N launcher count kernel-regex"
mkdir -p gpurun_out
TAG=${TAG:-r2}
while read -r robot alg dt n launcher count kre; do
  [ -z "$robot" ] && continue
  lt=${launcher}; [ "$lt" = "-" ] && lt=""
  base=gpurun_out/prof_${TAG}_${robot}_${alg}_${dt}_${n}${lt:+_$lt}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:${kre:-Knot_} -c ${count:-1} -o $base -f \
      python tools/profile_kernel.py --robot $robot --alg $alg --dtype $dt --n $n --launches 2 ${lt:+--launcher $lt} > $base.log 2>&1
  ncu -i $base.ncu-rep --page raw --csv > $base.raw.csv 2>/dev/null
  ncu -i $base.ncu-rep --page details --csv > $base.details.csv 2>/dev/null
  ncu -i $base.ncu-rep --page source --csv --print-source sass > $base.sass.csv 2>/dev/null
  gzip -f $base.sass.csv
  sz=$(stat -c %s $base.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 12000000 ]; then rm -f $base.ncu-rep; fi
done <<< "${PROFILE_LIST}"
du -sh gpurun_out
