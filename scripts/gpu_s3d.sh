#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s3d
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
timeout -s KILL 600 python bench.py > gpurun_out/${T}_bench.log 2>&1
tail -n 3 gpurun_out/${T}_tests.log; tail -1 gpurun_out/${T}_build.log; python -c "
import json; d=json.loads(open('gpurun_out/${T}_bench.log').read().strip().splitlines()[-1]); print(round(d['value']), d['ms_per_step'], d['e2e'], d['clocks']['sm_mhz'])"
