#!/bin/bash
# ring finalize determinism: A = current, E1 = loads consumed before the empty arrive, E2 = consumer barrier per row
cd "$GRAFT_REPO_ROOT"
L=paper_2410_10989_b200/lib
for v in A E1 E2 A E1 E2; do
  cp $L/ab/lib$v.so $L/libliger_b200.so
  echo "== $v" >> gpurun_out/r2g_ring.log
  timeout 600 python scripts/determinism_stage.py 2>&1 | grep -c '"z"' >> gpurun_out/r2g_ring.log
done
cat gpurun_out/r2g_ring.log
