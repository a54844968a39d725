#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s3i
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for cfg in "" "X --chunk-rows 4096" "" "X --chunk-rows 4096"; do
  if [ "${cfg:0:1}" = "X" ]; then ARGS="${cfg:2}"; ENVV=""; else ARGS=""; ENVV="$cfg"; fi
  echo "== $cfg" >> gpurun_out/${T}_bench.log
  env $ENVV timeout -s KILL 300 python bench.py --steps 30 --no-cpu-baseline $ARGS 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], {k: round(v,3) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['peak_mem']['peak_extra_minus_outputs'])" >> gpurun_out/${T}_bench.log 2>&1
done
cat gpurun_out/${T}_bench.log
