#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s2u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
timeout -s KILL 300 python bench_kernels.py --reps 20 > gpurun_out/${T}_kernels.log 2>&1
timeout -s KILL 300 python bench.py --config cfg4 --steps 20 --no-cpu-baseline > gpurun_out/${T}_bench_cfg4.log 2>&1
tail -n 4 gpurun_out/${T}_tests.log; grep summary gpurun_out/${T}_kernels.log; tail -c 1500 gpurun_out/${T}_bench_cfg4.log
