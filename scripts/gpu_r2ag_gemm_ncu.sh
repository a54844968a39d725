#!/bin/bash
# ncu --set full with source-level sampling of one logits GEMM and one backward GEMM launch (cfg2)
cd "$GRAFT_REPO_ROOT"
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:gemm2_kernel -s 8 -c 2 \
  -o gpurun_out/r2ag_gemm python scripts/profile_flce.py --steps 2 > gpurun_out/r2ag_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/r2ag_gemm.ncu-rep --page source --csv --print-source sass > gpurun_out/r2ag_sass.csv 2>&1
ncu -i gpurun_out/r2ag_gemm.ncu-rep --page details --csv > gpurun_out/r2ag_details.csv 2>&1
ls -la gpurun_out/r2ag_*
