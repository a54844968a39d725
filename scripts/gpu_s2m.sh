#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s2m
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_flce.py -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
timeout -s KILL 300 python bench.py --mode vocab --steps 20 > gpurun_out/${T}_bench_vocab.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:'gemm|ce_ring' -s 12 -c 12 -o gpurun_out/${T}_flce_step python scripts/profile_flce.py --steps 2 > gpurun_out/${T}_ncu_flce.log 2>&1
for K in rmsnorm_fwd rmsnorm_bwd colsum; do
  timeout -s KILL 300 ncu --set full --clock-control none -k regex:$K -c 1 -o gpurun_out/${T}_$K python bench_kernels.py --reps 1 --only rmsnorm > /dev/null 2>&1
done
timeout -s KILL 300 ncu --set full --clock-control none -k regex:ce_ring -c 1 -o gpurun_out/${T}_ce_ring python bench_kernels.py --reps 1 --only cross > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none -k regex:'rope|glu' -c 4 -o gpurun_out/${T}_rope_glu python bench_kernels.py --reps 1 --only rope,swiglu > /dev/null 2>&1
tail -n 3 gpurun_out/${T}_tests.log; tail -c 400 gpurun_out/${T}_bench_vocab.log; ls gpurun_out | grep $T
