#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep > gpurun_out/bench_r3.json 2> gpurun_out/bench_r3.err; tail -1 gpurun_out/bench_r3.json | cut -c1-400
SKIP_LAUNCHES=1 TAG=r3 PROFILE_LIST="chain7 gradFD f64 1048576
quad12 gradFD f64 1048576
humanoid30 gradFD f64 131072" bash tools/gpu_profile.sh > /dev/null 2>&1
RBD_TUNING='{"map": "ws", "maps": ["ws"], "warps": 8, "minb": 2}' SKIP_LAUNCHES=1 TAG=r3ws PROFILE_LIST="chain7 gradFD f64 1048576" bash tools/gpu_profile.sh > /dev/null 2>&1
ls gpurun_out | grep r3
