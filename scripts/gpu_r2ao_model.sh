#!/bin/bash
# model-level training step (Llama-3-8B-shaped decoder, 2 and 4 layers): stock HF vs upstream Liger vs this library
cd "$GRAFT_REPO_ROOT"
timeout 1200 python scripts/model_step_bench.py --layers 2 > gpurun_out/r2ao_model_l2.jsonl 2>&1
timeout 1200 python scripts/model_step_bench.py --layers 4 > gpurun_out/r2ao_model_l4.jsonl 2>&1
cat gpurun_out/r2ao_model_l2.jsonl gpurun_out/r2ao_model_l4.jsonl | grep -v summary
