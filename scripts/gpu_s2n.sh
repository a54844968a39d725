#!/bin/bash
# Profile captures summarised ON the box (raw .ncu-rep files exceed the 64 MiB return limit).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
T=s2n
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none -k regex:'gemm|ce_ring' -s 12 -c 12 -o /tmp/${T}_flce_step python scripts/profile_flce.py --steps 2 > gpurun_out/${T}_ncu_flce.log 2>&1
python scripts/profile_json.py /tmp/${T}_flce_step.ncu-rep gpurun_out/prof/r01_flce_step > /dev/null 2>&1
python scripts/ncu_summary.py report /tmp/${T}_flce_step.ncu-rep > gpurun_out/prof/r01_flce_step_full.md 2>&1
for K in rmsnorm_fwd rmsnorm_bwd colsum; do
  timeout -s KILL 300 ncu --set full --clock-control none -k regex:$K -c 1 -o /tmp/${T}_$K python bench_kernels.py --reps 1 --only rmsnorm > /dev/null 2>&1
  python scripts/ncu_summary.py report /tmp/${T}_$K.ncu-rep > gpurun_out/prof/r01_$K.md 2>&1
done
timeout -s KILL 300 ncu --set full --clock-control none -k regex:ce_ring -c 1 -o /tmp/${T}_ce_ring python bench_kernels.py --reps 1 --only cross > /dev/null 2>&1
python scripts/ncu_summary.py report /tmp/${T}_ce_ring.ncu-rep > gpurun_out/prof/r01_ce_ring.md 2>&1
timeout -s KILL 300 ncu --set full --clock-control none -k regex:'rope|glu' -c 4 -o /tmp/${T}_rope_glu python bench_kernels.py --reps 1 --only rope,swiglu > /dev/null 2>&1
python scripts/ncu_summary.py report /tmp/${T}_rope_glu.ncu-rep > gpurun_out/prof/r01_rope_glu.md 2>&1
cp /tmp/${T}_rmsnorm_bwd.ncu-rep gpurun_out/ 2>/dev/null
ls -la gpurun_out/prof; head -30 gpurun_out/prof/r01_flce_step.md
