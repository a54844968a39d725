#!/bin/bash
# round-2: segmented fp32 accumulation -- probe, full GPU suite, N=1 bench line
cd "$GRAFT_REPO_ROOT"
timeout 600 python scripts/probe_tc_accum.py > gpurun_out/r2d_probe.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 -p no:cacheprovider > gpurun_out/r2d_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2d_gputests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2d_bench_n1.jsonl 2> gpurun_out/r2d_bench_n1.err
grep flce_fp32 gpurun_out/r2d_probe.jsonl; tail -3 gpurun_out/r2d_gputests.log; head -c 400 gpurun_out/r2d_bench_n1.jsonl
