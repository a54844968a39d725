#!/bin/bash
# A/B: RoPE, A = semi-persistent token-range kernel, R2/R4/R8 = one CTA per 2/4/8 tokens (all loads first)
cd "$GRAFT_REPO_ROOT"
L=paper_2410_10989_b200/lib
for r in 1 2; do for v in R1 R2; do
  cp $L/ab/lib$v.so $L/libliger_b200.so
  echo "$v kvl: $(python scripts/kernel_vs_liger.py --only rope 2>&1 | tail -1)" >> gpurun_out/r2x_ab.log
  echo "$v bk: $(python bench_kernels.py --only rope 2>&1 | tail -1)" >> gpurun_out/r2x_ab.log
done; done
cp $L/ab/libR2.so $L/libliger_b200.so
timeout 600 python -m pytest tests/test_gpu_rowops.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/r2x_ab.log
cat gpurun_out/r2x_ab.log
