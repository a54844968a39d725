#!/bin/bash
# round-2 re-entry check: full -m gpu suite + smoke + N=1 bench line
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2b_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=25 -p no:cacheprovider > gpurun_out/r2b_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2b_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench_n1.jsonl 2> gpurun_out/r2b_bench_n1.err
tail -3 gpurun_out/r2b_gputests.log; tail -2 gpurun_out/r2b_smoke.log; tail -c 1500 gpurun_out/r2b_bench_n1.jsonl
