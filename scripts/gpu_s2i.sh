#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s2i
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
for cfg in "" "LK_NORM_BWD_THREADS=512" "LK_NORM_NO_BF16_FAST=1" "LK_NORM_BWD_SLOTS=6"; do
  echo "== $cfg" >> gpurun_out/${T}_kernels.log
  env $cfg timeout -s KILL 120 python bench_kernels.py --reps 20 --only rmsnorm >> gpurun_out/${T}_kernels.log 2>&1
done
timeout -s KILL 300 python bench_kernels.py --reps 20 > gpurun_out/${T}_kernels_all.log 2>&1
timeout -s KILL 600 python bench.py > gpurun_out/${T}_bench.log 2>&1
tail -n 2 gpurun_out/${T}_tests.log; grep -E "==|summary" gpurun_out/${T}_kernels.log gpurun_out/${T}_kernels_all.log; tail -c 600 gpurun_out/${T}_bench.log
