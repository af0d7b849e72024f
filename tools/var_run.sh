VARIANTS=tools/variants_h30.txt bash tools/variants.sh time humanoid30 gradFD f64 262144 2>&1 | cut -c 1-140
