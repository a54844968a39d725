#!/bin/bash
# model-level training step after the kept-row FLCE and the 3-chunk plan (2 and 4 layers), all three implementations
cd "$GRAFT_REPO_ROOT"
timeout 1200 python scripts/model_step_bench.py --layers 2 > gpurun_out/r2bg_model_l2.jsonl 2>&1
timeout 1200 python scripts/model_step_bench.py --layers 4 > gpurun_out/r2bg_model_l4.jsonl 2>&1
cat gpurun_out/r2bg_model_l2.jsonl gpurun_out/r2bg_model_l4.jsonl | grep -v summary
