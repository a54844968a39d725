#!/bin/bash
# A/B of the bf16 FLCE: A = before piece-addressed operand modes, B = with them
cd "$GRAFT_REPO_ROOT"
L=paper_2410_10989_b200/lib
for r in 1 2 3; do for v in A B; do
  cp $L/ab/lib$v.so $L/libliger_b200.so
  echo "$v: $(python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), {k: round(v, 3) for k, v in d["roofline"]["stage_ms_per_step"].items()}, d["clocks"]["sm_mhz"])')" >> gpurun_out/r2ae_ab.log
done; done
cat gpurun_out/r2ae_ab.log
