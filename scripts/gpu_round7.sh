#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests7.log
LK_NORM_NO_TMA=1 timeout -s KILL 300 python -m pytest tests/test_gpu_rowops.py -q -k rmsnorm --timeout 200 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests7_normfb.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests7_normfb.log
timeout -s KILL 600 python bench.py > gpurun_out/bench7.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench7.log
timeout -s KILL 300 python bench_kernels.py --reps 20 > gpurun_out/kernels7.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm2_kernel -s 4 -c 2 -o gpurun_out/r01_gemm_v6 python scripts/profile_flce.py --steps 2 > gpurun_out/ncu_gemm7.log 2>&1
tail -2 gpurun_out/gpu_tests7.log gpurun_out/gpu_tests7_normfb.log gpurun_out/bench7.log gpurun_out/kernels7.log
