#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s2v
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_rowops.py tests/test_converge.py -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
timeout -s KILL 300 python bench_kernels.py --reps 20 --only layernorm,rmsnorm > gpurun_out/${T}_kernels.log 2>&1
tail -n 4 gpurun_out/${T}_tests.log; grep summary gpurun_out/${T}_kernels.log
