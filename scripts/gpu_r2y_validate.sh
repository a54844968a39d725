#!/bin/bash
# validate chunked GLU + RoPE: full GPU suite, smoke, kernel bench (cold/steady), kernel-level vs Liger
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2y_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2y_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1
timeout 600 python bench_kernels.py --reps 20 > gpurun_out/r2y_kernels.jsonl 2>&1
timeout 600 python scripts/kernel_vs_liger.py > gpurun_out/r2y_kernel_vs_liger.jsonl 2>&1
tail -2 gpurun_out/r2y_gputests.log; tail -1 gpurun_out/r2y_smoke.log; tail -1 gpurun_out/r2y_kernels.jsonl; tail -1 gpurun_out/r2y_kernel_vs_liger.jsonl
