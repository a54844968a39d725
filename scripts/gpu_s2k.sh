#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s2k
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_rowops.py -q -rf --timeout 200 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
for cfg in "" "LK_NORM_BWD_THREADS=128" "LK_NORM_BWD_THREADS=128 LK_NORM_BWD_SLOTS=3"; do
  echo "== $cfg" >> gpurun_out/${T}_kernels.log
  env $cfg timeout -s KILL 120 python bench_kernels.py --reps 20 --only rmsnorm >> gpurun_out/${T}_kernels.log 2>&1
done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:'rmsnorm|colsum' --csv python bench_kernels.py --reps 2 --only rmsnorm > gpurun_out/${T}_ncu_list.csv 2>&1
tail -n 2 gpurun_out/${T}_tests.log; grep -E "==|rmsnorm" gpurun_out/${T}_kernels.log | cut -c1-60,200-330
