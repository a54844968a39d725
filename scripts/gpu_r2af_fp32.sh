#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_gpu_parity_headline.py tests/test_gpu_gemm.py tests/test_converge.py -m gpu -q -p no:cacheprovider -k "fp32 or gemm or converge" > gpurun_out/r2af_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2af_tests.log
tail -3 gpurun_out/r2af_tests.log
