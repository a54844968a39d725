#!/bin/bash
# A/B: column-sum kernel (A = LN bwd 256 threads, B = 128 threads)
cd "$GRAFT_REPO_ROOT"
L=paper_2410_10989_b200/lib
for r in 1 2; do for v in A B; do
  cp $L/ab/lib$v.so $L/libliger_b200.so
  echo "$v: $(python bench_kernels.py --only layernorm --reps 30 2>&1 | tail -1)" >> gpurun_out/r2n_ab.log
done; done
cp $L/ab/libB.so $L/libliger_b200.so
timeout 600 python -m pytest tests/test_gpu_rowops.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/r2n_ab.log
cat gpurun_out/r2n_ab.log
