#!/bin/bash
# ring release fix: stage determinism (24 repeats), full GPU suite, N=1 bench, CE kernel bench
cd "$GRAFT_REPO_ROOT"
timeout 600 python scripts/determinism_stage.py > gpurun_out/r2h_det.log 2>&1
echo "differing repeats: $(grep -c '"z"' gpurun_out/r2h_det.log)" >> gpurun_out/r2h_det.log
timeout 1500 python -m pytest tests -m gpu -q --durations=10 -p no:cacheprovider > gpurun_out/r2h_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2h_gputests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2h_bench_n1.jsonl 2> gpurun_out/r2h_bench_n1.err
timeout 300 python bench_kernels.py --only cross_entropy > gpurun_out/r2h_ce.jsonl 2>&1
tail -1 gpurun_out/r2h_det.log; tail -3 gpurun_out/r2h_gputests.log; head -c 300 gpurun_out/r2h_bench_n1.jsonl; tail -1 gpurun_out/r2h_ce.jsonl
