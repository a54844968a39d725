#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 120 python scripts/gemm_probe.py > gpurun_out/gemm_probe5.log 2>&1; echo "probe rc=$?" >> gpurun_out/gemm_probe5.log
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests5.log
LK_NO_TMA_EPILOGUE=1 LK_CTA_GROUP=1 timeout -s KILL 600 python -m pytest tests/test_gpu_flce.py tests/test_gpu_gemm.py -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests5_legacy.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests5_legacy.log
timeout -s KILL 600 python bench.py > gpurun_out/bench5.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench5.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm2_kernel -s 4 -c 2 -o gpurun_out/r01_gemm_v4 python scripts/profile_flce.py --steps 2 > gpurun_out/ncu_gemm5.log 2>&1
tail -2 gpurun_out/gemm_probe5.log gpurun_out/gpu_tests5.log gpurun_out/gpu_tests5_legacy.log gpurun_out/bench5.log
