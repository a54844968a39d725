#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s2l
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_tests.log
timeout -s KILL 600 python bench.py > gpurun_out/${T}_bench.log 2>&1
LK_FLCE_SEPARATE_CAST=1 LK_FLCE_FINALIZE_BLOCK=1 timeout -s KILL 600 python bench.py --steps 20 > gpurun_out/${T}_bench_old.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/${T}_ncu_launch.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:'gemm|ce_ring' -s 8 -c 4 -o gpurun_out/${T}_flce python scripts/profile_flce.py --steps 2 > gpurun_out/${T}_ncu_flce.log 2>&1
tail -n 2 gpurun_out/${T}_tests.log; tail -c 900 gpurun_out/${T}_bench.log; echo; grep -o '"value": [0-9.]*' gpurun_out/${T}_bench_old.log | head -1
