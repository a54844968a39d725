#!/bin/bash
# round-2: tcgen05 fp32-accumulation probe (fp32 split FLCE parity), bandwidth kernels cold+steady,
# ncu DRAM bytes + duration per bandwidth-kernel launch
cd "$GRAFT_REPO_ROOT"
timeout 600 python scripts/probe_tc_accum.py > gpurun_out/r2c_probe.jsonl 2>&1
timeout 600 python bench_kernels.py --reps 20 > gpurun_out/r2c_kernels.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/r2c_kernels_ncu.csv python bench_kernels.py --reps 1 > /dev/null 2>&1
echo "ncu rc=$?"
cat gpurun_out/r2c_probe.jsonl; tail -1 gpurun_out/r2c_kernels.jsonl
