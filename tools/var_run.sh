timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "humanoid30" 2>&1 | tail -2
for dt in f64 f32; do python tools/time_kernel.py --robot humanoid30 --alg gradFD --dtype $dt --n 65536 262144 | cut -c1-150; done
