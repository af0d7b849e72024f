#!/bin/bash
# SASS opcode histogram of one kernel: tools/sass_hist.sh <file.so|.o> <symbol-substring>
cuobjdump -sass "$1" 2>/dev/null | awk -v pat="$2" '/Function :/ {on = index($0, pat) > 0} on' \
  | grep -oP '^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[T0-9]+\s+)?\K[A-Z0-9]+' | sort | uniq -c | sort -rn | head -${3:-25}
