while read -r v; do
  key=x$(printf '%s' "$v" | md5sum | cut -c1-7)
  for i in 1 2; do for r in chain7 quad12; do
    echo "$v"; RBD_PARTIAL_BUILD=1 RBD_TUNING="$v" RBD_BUILD_KEY=$key timeout 300 python tools/small_n.py $r gradFD,ID f64 16,128,256 2>&1 | grep "{"
  done; done
done < tools/experiments/variants_wsincos.txt
