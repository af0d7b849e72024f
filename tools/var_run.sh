timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for alg in gradFD gradID; do for dt in f64 f32; do python tools/time_kernel.py --robot humanoid30 --alg $alg --dtype $dt --n 262144 | cut -c1-150; done; done
