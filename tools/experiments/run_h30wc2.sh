while read -r v; do
  key=x$(printf '%s' "$v" | md5sum | cut -c1-7)
  echo "$v"; RBD_PARTIAL_BUILD=1 RBD_TUNING="$v" RBD_BUILD_KEY=$key timeout 300 python tools/small_n.py humanoid30 gradFD f64 16,128,256,1024 2>&1 | grep "{"
done < tools/experiments/variants_h30wc2.txt
timeout 300 python tools/small_n.py humanoid30 gradFD f64 16,128,256,1024 2>&1 | grep "{"
