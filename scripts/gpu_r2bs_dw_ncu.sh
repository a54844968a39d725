#!/bin/bash
# ncu --set full + source sampling of the dW-shaped GEMM at K=2560 and K=10240 (the per-pass cost)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2bs
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:gemm2_kernel -s 1 -c 1 \
  -o ${O}_k2560 python scripts/dw_gemm_once.py 2560 > ${O}_ncu.log 2>&1
echo "rc=$?"
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:gemm2_kernel -s 1 -c 1 \
  -o ${O}_k10240 python scripts/dw_gemm_once.py 10240 >> ${O}_ncu.log 2>&1
echo "rc=$?"
for k in 2560 10240; do
  ncu -i ${O}_k$k.ncu-rep --page source --csv --print-source sass > ${O}_k${k}_sass.csv 2>&1
  ncu -i ${O}_k$k.ncu-rep --page details --csv > ${O}_k${k}_details.csv 2>&1
done
ls -la gpurun_out/ | grep r2bs
