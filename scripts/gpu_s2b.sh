#!/bin/bash
# Ring kernels (RMSNorm / standalone CE): parity vs other paths + oracle, kernel bench, ncu.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s2b_build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_ce.py -q -rf --timeout 200 --timeout-method=thread -p no:cacheprovider > gpurun_out/s2b_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s2b_tests.log
timeout -s KILL 300 python bench_kernels.py --reps 20 > gpurun_out/s2b_kernels.log 2>&1; echo "kernels rc=$?" >> gpurun_out/s2b_kernels.log
LK_NORM_IMPL=warp LK_CE_IMPL=block timeout -s KILL 300 python bench_kernels.py --reps 20 --only rmsnorm,cross > gpurun_out/s2b_kernels_old.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:'ring' -c 4 -o gpurun_out/s2b_ring python bench_kernels.py --reps 1 --only rmsnorm,cross > gpurun_out/s2b_ncu.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/s2b_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s2b_gpu_tests.log
tail -n 3 gpurun_out/s2b_tests.log gpurun_out/s2b_gpu_tests.log; cat gpurun_out/s2b_kernels.log gpurun_out/s2b_kernels_old.log | grep summary
