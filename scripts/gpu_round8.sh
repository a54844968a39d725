#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests8.log
LK_NORM_NO_FAST=1 timeout -s KILL 300 python -m pytest tests/test_gpu_rowops.py -q -k rmsnorm --timeout 200 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests8_normfb.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests8_normfb.log
timeout -s KILL 600 python bench.py > gpurun_out/bench8.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench8.log
timeout -s KILL 300 python bench_kernels.py --reps 20 > gpurun_out/kernels8.log 2>&1
tail -2 gpurun_out/gpu_tests8.log gpurun_out/gpu_tests8_normfb.log gpurun_out/bench8.log gpurun_out/kernels8.log
