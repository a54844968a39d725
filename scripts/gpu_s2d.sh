#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s2d
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_ce.py -q -rf --timeout 200 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
timeout -s KILL 300 python bench_kernels.py --reps 20 > gpurun_out/${T}_kernels.log 2>&1
for K in rmsnorm_fwd_ring rmsnorm_bwd_ring ce_ring; do
  O=rmsnorm; [ $K = ce_ring ] && O=cross
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/${T}_$K python bench_kernels.py --reps 1 --only $O > gpurun_out/${T}_ncu_$K.log 2>&1
done
tail -n 2 gpurun_out/${T}_tests.log; grep summary gpurun_out/${T}_kernels.log
