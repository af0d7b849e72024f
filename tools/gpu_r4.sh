mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
TAG=r4 SKIP_LAUNCHES=1 PROFILE_LIST="chain7 gradFD f64 1048576
quad12 gradFD f64 1048576" bash tools/gpu_profile.sh > /dev/null 2>&1
ls gpurun_out | head -30
