#!/bin/bash
# new default plan above 16384 tokens: cfg5 one-GPU parity test, plan tests, cfg5 bench line
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_flce.py -m gpu -q -x -k "cfg5 or finalize or cfg2 or cfg4" -p no:cacheprovider > gpurun_out/r2p_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2p_tests.log
timeout 600 python bench.py --config cfg5 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r2p_bench_cfg5_n1.jsonl 2>&1
tail -3 gpurun_out/r2p_tests.log; head -c 300 gpurun_out/r2p_bench_cfg5_n1.jsonl
