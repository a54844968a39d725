#!/bin/bash
# Same-box A/B of two prebuilt library variants: scripts/ab.sh "<bench args>" [rounds]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
L=paper_2410_10989_b200/lib
for r in $(seq 1 ${2:-2}); do
  for v in A B; do
    cp $L/ab/lib$v.so $L/libliger_b200.so
    echo "$v: $(python bench_kernels.py $1 2>&1 | tail -1)"
  done
done
