#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 120 python scripts/gemm_probe.py > gpurun_out/gemm_probe4.log 2>&1; echo "probe rc=$?" >> gpurun_out/gemm_probe4.log
if grep -q "cg2: exact=True" gpurun_out/gemm_probe4.log; then
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests4.log
timeout -s KILL 600 python bench.py > gpurun_out/bench4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench4.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm2_kernel -s 4 -c 2 -o gpurun_out/r01_gemm_v3 python scripts/profile_flce.py --steps 2 > gpurun_out/ncu_gemm4.log 2>&1
fi
tail -3 gpurun_out/gemm_probe4.log gpurun_out/gpu_tests4.log gpurun_out/bench4.log
