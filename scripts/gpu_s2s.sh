#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s2s
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
timeout -s KILL 600 python bench.py > gpurun_out/${T}_bench.log 2>&1
tail -n 4 gpurun_out/${T}_tests.log; tail -c 300 gpurun_out/${T}_bench.log
