while read -r v; do
  key=x$(printf '%s' "$v" | md5sum | cut -c1-7)
  echo "$v"; RBD_PARTIAL_BUILD=1 RBD_TUNING="$v" RBD_BUILD_KEY=$key timeout 300 python tools/small_n.py chain7 gradFD,ID f64 16,128,1024 2>&1 | grep "{" | cut -c1-120
done < tools/experiments/variants_c7ws.txt
