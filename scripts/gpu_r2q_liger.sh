#!/bin/bash
# same-box comparison with upstream Liger-Kernel 0.8.0 (Triton + cuBLAS) and torch eager, round-2 library
cd "$GRAFT_REPO_ROOT"
timeout 1200 python scripts/compare_liger.py --reps 10 > gpurun_out/r2q_vs_liger.jsonl 2> gpurun_out/r2q_vs_liger.err
tail -c 2000 gpurun_out/r2q_vs_liger.jsonl
