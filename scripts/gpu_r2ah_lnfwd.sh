#!/bin/bash
# A/B: LayerNorm fwd, A = row unpacked to fp32 registers, B = row kept as raw vectors
cd "$GRAFT_REPO_ROOT"
L=paper_2410_10989_b200/lib
for r in 1 2; do for v in A B; do
  cp $L/ab/lib$v.so $L/libliger_b200.so
  echo "$v kvl: $(python scripts/kernel_vs_liger.py --only layernorm 2>&1 | tail -1)" >> gpurun_out/r2ah_ab.log
  echo "$v bk: $(python bench_kernels.py --only layernorm 2>&1 | tail -1)" >> gpurun_out/r2ah_ab.log
done; done
cat gpurun_out/r2ah_ab.log
