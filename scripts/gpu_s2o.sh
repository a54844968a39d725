#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
T=s2o
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_flce.py tests/test_gpu_gemm.py -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
timeout -s KILL 600 python bench.py > gpurun_out/${T}_bench.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none -k regex:'gemm|ce_ring' -s 12 -c 12 -o /tmp/${T}_flce_step python scripts/profile_flce.py --steps 2 > gpurun_out/${T}_ncu_flce.log 2>&1
python scripts/profile_json.py /tmp/${T}_flce_step.ncu-rep gpurun_out/prof/${T}_flce_step > /dev/null 2>&1
tail -n 3 gpurun_out/${T}_tests.log; tail -n 2 gpurun_out/${T}_build.log; cat gpurun_out/prof/${T}_flce_step.md; python -c "
import json; d=json.loads(open('gpurun_out/${T}_bench.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['stage_ms_per_step'], d['peak_mem'], d['clocks'], d['e2e']['value'])"
