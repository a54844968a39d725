#!/bin/bash
# ncu --set full: LayerNorm fwd/bwd, RMSNorm bwd + its column sum (cfg3, 8192 x 4096 bf16)
cd "$GRAFT_REPO_ROOT"
for k in layernorm_bwd layernorm_fwd rmsnorm_bwd colsum; do
  only=layernorm; [[ $k == rmsnorm_bwd || $k == colsum ]] && only=rmsnorm
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/r2m_$k \
    python bench_kernels.py --reps 1 --only $only > gpurun_out/r2m_${k}_ncu.log 2>&1
  python scripts/ncu_summary.py report gpurun_out/r2m_$k.ncu-rep > gpurun_out/r2m_$k.md 2>&1
  ncu -i gpurun_out/r2m_$k.ncu-rep --page details --csv > gpurun_out/r2m_${k}_details.csv 2>&1
done
ls -la gpurun_out/r2m_*
