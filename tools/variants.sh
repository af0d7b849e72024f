#!/bin/bash
# build (here) or time (on the GPU box) a list of tuning variants
# usage: tools/variants.sh build|time robot alg dtype N...
# ALGS / DTYPES (build): comma lists -> a partial library of those entries
# (RBD_PARTIAL_BUILD=1 is then needed to load it; never use it for the
# default tuning "{}", whose build key is the product's)
mode=$1; robot=$2; alg=$3; dt=$4; shift 4
while read -r v; do
  [ -z "$v" ] && continue
  export RBD_BUILD_KEY=x$(printf '%s' "$v" | md5sum | cut -c1-7)
  if [ "$mode" = build ]; then
    RBD_TUNING="$v" python -c "
import sys; sys.path.insert(0,'.')
from paper_2109_06976_b200 import models, kernels, codegen
algs = '${ALGS:-}'.split(',') if '${ALGS:-}' else codegen.ALGORITHMS
dts = '${DTYPES:-}'.split(',') if '${DTYPES:-}' else codegen.DTYPES
kernels.compile_library(models.load('$robot'), algorithms=algs, dtypes=dts)" || echo "build failed $v"
  else
    RBD_PARTIAL_BUILD=1 RBD_TUNING="$v" timeout 300 python tools/time_kernel.py --robot $robot --alg $alg --dtype $dt --n "$@"
  fi
done < ${VARIANTS:?set VARIANTS to a file of tuning JSON lines (tools/experiments/)}
