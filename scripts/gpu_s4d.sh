#!/bin/bash
# ncu --set full of the standalone CE ring kernel (bf16 8192 x 128256); raw + SASS source pages to CSV on the box
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s4d
timeout -s KILL 400 ncu --set full --clock-control none -k regex:ce_ring -c 1 -o /tmp/${T}_ce \
  python bench_kernels.py --reps 1 --only cross > gpurun_out/${T}_ncu.log 2>&1
timeout 120 ncu -i /tmp/${T}_ce.ncu-rep --page raw --csv > gpurun_out/${T}_ce_raw.csv 2>&1
timeout 120 ncu -i /tmp/${T}_ce.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_ce_sass.csv 2>&1
ls -la gpurun_out/${T}_*
