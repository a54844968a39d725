#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python scripts/kernel_vs_liger.py --reps 20 > gpurun_out/r2s_kernel_vs_liger.jsonl 2> gpurun_out/r2s_kvl.err
cat gpurun_out/r2s_kernel_vs_liger.jsonl; tail -5 gpurun_out/r2s_kvl.err
