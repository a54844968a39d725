#!/bin/bash
# round-2: cfg4 determinism A (before segmented accumulation) vs B (after); kernel bench on B
cd "$GRAFT_REPO_ROOT"
L=paper_2410_10989_b200/lib
for v in A B A B; do
  cp $L/ab/lib$v.so $L/libliger_b200.so
  echo "== $v" >> gpurun_out/r2e_det.log
  timeout 600 python scripts/determinism_cfg4.py >> gpurun_out/r2e_det.log 2>&1
done
timeout 600 python bench_kernels.py --reps 20 > gpurun_out/r2e_kernels.jsonl 2>&1
cat gpurun_out/r2e_det.log; tail -2 gpurun_out/r2e_kernels.jsonl
