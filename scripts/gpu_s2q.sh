#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s2q
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
timeout -s KILL 600 python bench.py > gpurun_out/${T}_bench.log 2>&1
timeout -s KILL 300 python bench.py --impl reference > gpurun_out/${T}_bench_ref.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/${T}_ncu_launch.log 2>&1
tail -n 3 gpurun_out/${T}_tests.log; tail -n 1 gpurun_out/${T}_build.log
