#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_flce.py -m gpu -q -p no:cacheprovider -k "fp32 or slices" > gpurun_out/r2ai_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2ai_tests.log
tail -15 gpurun_out/r2ai_tests.log
