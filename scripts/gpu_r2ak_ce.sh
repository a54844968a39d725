#!/bin/bash
# A/B: standalone CE ring pass 1, A = chained max / sum, B = tree max + per-vector accumulators
cd "$GRAFT_REPO_ROOT"
L=paper_2410_10989_b200/lib
for r in 1 2 3; do for v in A B; do
  cp $L/ab/lib$v.so $L/libliger_b200.so
  echo "$v: $(python bench_kernels.py --only cross_entropy 2>&1 | tail -1)" >> gpurun_out/r2ak_ab.log
done; done
cp $L/ab/libB.so $L/libliger_b200.so
timeout 900 python -m pytest tests/test_gpu_ce.py tests/test_gpu_flce.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/r2ak_ab.log
cat gpurun_out/r2ak_ab.log
