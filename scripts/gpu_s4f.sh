#!/bin/bash
# ncu --set full of the LayerNorm backward (8192 x 4096 bf16): raw + SASS pages to CSV on the box
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s4f
timeout -s KILL 400 ncu --set full --clock-control none -k regex:layernorm_bwd -c 1 -o /tmp/${T}_ln \
  python bench_kernels.py --reps 1 --only layernorm > gpurun_out/${T}_ncu.log 2>&1
timeout 120 ncu -i /tmp/${T}_ln.ncu-rep --page raw --csv > gpurun_out/${T}_ln_raw.csv 2>&1
timeout 120 ncu -i /tmp/${T}_ln.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_ln_sass.csv 2>&1
python scripts/ncu_summary.py report /tmp/${T}_ln.ncu-rep > gpurun_out/${T}_ln.md 2>&1
ls -la gpurun_out/${T}_*
