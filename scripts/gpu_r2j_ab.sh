#!/bin/bash
# A/B of norm backward partial reductions: C1 = per-CTA partials, C4 = clusters of 4, C2 = clusters of 2
cd "$GRAFT_REPO_ROOT"
L=paper_2410_10989_b200/lib
for r in 1 2; do for v in C1 C4 C2; do
  cp $L/ab/lib$v.so $L/libliger_b200.so
  echo "$v: $(python bench_kernels.py --only rmsnorm,layernorm --reps 30 2>&1 | tail -1)" >> gpurun_out/r2j_ab.log
done; done
cp $L/ab/libC2.so $L/libliger_b200.so
timeout 600 python -m pytest tests/test_gpu_rowops.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/r2j_ab.log
cat gpurun_out/r2j_ab.log
