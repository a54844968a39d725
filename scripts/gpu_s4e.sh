#!/bin/bash
# kernel bench (all bandwidth kernels) + ncu summaries of the CE ring and the norm backward kernels
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
T=s4e
python bench_kernels.py --reps 30 > gpurun_out/prof/r01_kernels.jsonl 2>&1
timeout -s KILL 400 ncu --set full --clock-control none -k regex:ce_ring -c 1 -o /tmp/${T}_ce_ring python bench_kernels.py --reps 1 --only cross > /dev/null 2>&1
python scripts/ncu_summary.py report /tmp/${T}_ce_ring.ncu-rep > gpurun_out/prof/r01_ce_ring.md 2>&1
timeout -s KILL 400 ncu --set full --clock-control none -k regex:'layernorm_bwd|rmsnorm_bwd' -c 2 -o /tmp/${T}_norm_bwd python bench_kernels.py --reps 1 --only rmsnorm,layernorm > /dev/null 2>&1
python scripts/ncu_summary.py report /tmp/${T}_norm_bwd.ncu-rep > gpurun_out/prof/r01_norm_bwd.md 2>&1
tail -1 gpurun_out/prof/r01_kernels.jsonl; ls -la gpurun_out/prof
