#!/bin/bash
# ncu --set full of the standalone CE ring and the FLCE finalize: pipe utilisation (is the ring MUFU-bound?)
cd "$GRAFT_REPO_ROOT"
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:ce_ring_kernel -c 1 \
  -o gpurun_out/r2aj_ce python bench_kernels.py --reps 1 --only cross_entropy > gpurun_out/r2aj_ncu.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:ce_ring_kernel -s 2 -c 1 \
  -o gpurun_out/r2aj_fin python scripts/profile_flce.py --steps 1 >> gpurun_out/r2aj_ncu.log 2>&1
for f in ce fin; do
  ncu -i gpurun_out/r2aj_$f.ncu-rep --page details --csv > gpurun_out/r2aj_${f}_details.csv 2>&1
  ncu -i gpurun_out/r2aj_$f.ncu-rep --page raw --csv > gpurun_out/r2aj_${f}_raw.csv 2>&1
done
ncu -i gpurun_out/r2aj_ce.ncu-rep --page source --csv --print-source sass > gpurun_out/r2aj_ce_sass.csv 2>&1
ls -la gpurun_out/r2aj_*
