#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s3a
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_flce.py -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
for cfg in "" "LK_EXP_EPI=2" ""; do
  echo "== $cfg" >> gpurun_out/${T}_bench.log
  env $cfg timeout -s KILL 300 python bench.py --steps 30 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], {k: round(v,3) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/${T}_bench.log 2>&1
done
timeout -s KILL 300 python bench.py --config cfg4 --steps 20 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('cfg4', round(d['value']), d['ms_per_step'], d['roofline']['step_tflops'], {k: round(v,3) for k,v in d['roofline']['stage_ms_per_step'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/${T}_bench.log 2>&1
tail -n 3 gpurun_out/${T}_tests.log; cat gpurun_out/${T}_bench.log
