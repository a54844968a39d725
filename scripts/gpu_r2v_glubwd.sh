#!/bin/bash
# A/B: GLU backward, A = grid-stride, U2/U4/U8 = one CTA per chunk of U x 256 vectors (forward chunked in all U*)
cd "$GRAFT_REPO_ROOT"
L=paper_2410_10989_b200/lib
for r in 1 2; do for v in A U2 U4 U8; do
  cp $L/ab/lib$v.so $L/libliger_b200.so
  echo "$v bk: $(python bench_kernels.py --only swiglu,geglu 2>&1 | tail -1)" >> gpurun_out/r2v_ab.log
done; done
cat gpurun_out/r2v_ab.log
