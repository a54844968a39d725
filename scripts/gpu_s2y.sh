#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s2y
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for cfg in "" "LK_LOGITS_PF=8" "LK_LOGITS_PF=16" "LK_LOGITS_PF=32" "" "LK_LOGITS_PF=16 LK_DX_PF=16"; do
  echo "== $cfg" >> gpurun_out/${T}_bench.log
  env $cfg timeout -s KILL 300 python bench.py --steps 30 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], {k: round(v,3) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/${T}_bench.log 2>&1
done
cat gpurun_out/${T}_bench.log
