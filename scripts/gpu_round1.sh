#!/bin/bash
# First GPU pass: GEMM probe, GPU tests, smoke, short bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 180 python scripts/gemm_probe.py > gpurun_out/gemm_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/gemm_probe.log
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 600 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -5 gpurun_out/gemm_probe.log gpurun_out/gpu_tests.log gpurun_out/smoke.log gpurun_out/bench.log
