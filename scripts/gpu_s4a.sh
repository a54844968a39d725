#!/bin/bash
# cfg2 vs cfg4 stage breakdown (logits GEMM+epilogue / finalize / backward GEMMs)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s4a
for ARGS in "--config cfg2" "--config cfg4"; do
  echo "== $ARGS" >> gpurun_out/${T}_bench.log
  timeout -s KILL 300 python bench.py --steps 20 --no-cpu-baseline $ARGS 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], {k: round(v,3) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['roofline']['achieved'])" >> gpurun_out/${T}_bench.log 2>&1
done
cat gpurun_out/${T}_bench.log
