#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s3h
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_rowops.py tests/test_converge.py -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
timeout -s KILL 300 python bench_kernels.py --reps 20 --only swiglu,geglu > gpurun_out/${T}_kernels.log 2>&1
timeout -s KILL 600 python bench.py --steps 30 > gpurun_out/${T}_bench.log 2>&1
tail -n 3 gpurun_out/${T}_tests.log; grep summary gpurun_out/${T}_kernels.log; python -c "
import json; d=json.loads(open('gpurun_out/${T}_bench.log').read().strip().splitlines()[-1]); print(round(d['value']), d['ms_per_step'], d['roofline']['stage_ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'])"
