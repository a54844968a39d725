#!/bin/bash
# chunk-size sweep at cfg2 (steady state, default weight-dtype accumulation)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s4c
for CR in 2048 4096 8192 2048 4096 8192; do
  echo "== chunk_rows $CR" >> gpurun_out/${T}_bench.log
  timeout -s KILL 300 python bench.py --steps 30 --no-cpu-baseline --chunk-rows $CR 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['peak_mem'])" >> gpurun_out/${T}_bench.log 2>&1
done
cat gpurun_out/${T}_bench.log
