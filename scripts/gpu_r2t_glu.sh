#!/bin/bash
# A/B: GLU kernels, A = grid-stride (2 vectors/thread), B = blocked (4 / 2 vectors per thread)
cd "$GRAFT_REPO_ROOT"
L=paper_2410_10989_b200/lib
for r in 1 2; do for v in A B; do
  cp $L/ab/lib$v.so $L/libliger_b200.so
  echo "$v kvl: $(python scripts/kernel_vs_liger.py --only swiglu 2>&1 | tail -1)" >> gpurun_out/r2t_ab.log
  echo "$v bk: $(python bench_kernels.py --only swiglu,geglu 2>&1 | tail -1)" >> gpurun_out/r2t_ab.log
done; done
cp $L/ab/libB.so $L/libliger_b200.so
timeout 600 python -m pytest tests/test_gpu_rowops.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/r2t_ab.log
cat gpurun_out/r2t_ab.log
