#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s2e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_rowops.py -q -rf --timeout 200 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
for cfg in "" "LK_NORM_FWD_THREADS=256" "LK_NORM_FWD_THREADS=64" "LK_NORM_BWD_THREADS=128" "LK_NORM_BWD_CTAS_PER_SM=1" "LK_NORM_IMPL=ring"; do
  echo "== $cfg" >> gpurun_out/${T}_kernels.log
  env $cfg timeout -s KILL 120 python bench_kernels.py --reps 20 --only rmsnorm >> gpurun_out/${T}_kernels.log 2>&1
done
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:rmsnorm -c 2 -o gpurun_out/${T}_cta python bench_kernels.py --reps 1 --only rmsnorm > gpurun_out/${T}_ncu.log 2>&1
tail -n 2 gpurun_out/${T}_tests.log; grep -E "==|summary" gpurun_out/${T}_kernels.log
