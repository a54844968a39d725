#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 200 python scripts/gemm_probe.py > gpurun_out/gemm_probe.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests3.log
timeout -s KILL 600 python bench.py > gpurun_out/bench3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench3.log
timeout -s KILL 300 python bench_kernels.py --reps 20 > gpurun_out/kernels3.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 4 -c 2 -o gpurun_out/r01_gemm_v2 python scripts/profile_flce.py --steps 2 > gpurun_out/ncu_gemm3.log 2>&1
tail -3 gpurun_out/gemm_probe.log gpurun_out/gpu_tests3.log gpurun_out/bench3.log gpurun_out/kernels3.log
