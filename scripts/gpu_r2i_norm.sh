#!/bin/bash
# cluster-reduced norm partials + cheaper ring release: row-op/CE tests, determinism, kernel bench
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_ce.py tests/test_gpu_flce.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2i_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2i_tests.log
timeout 600 python scripts/determinism_stage.py > gpurun_out/r2i_det.log 2>&1
echo "differing repeats: $(grep -c '"z"' gpurun_out/r2i_det.log)" >> gpurun_out/r2i_det.log
timeout 600 python bench_kernels.py --reps 20 > gpurun_out/r2i_kernels.jsonl 2>&1
tail -2 gpurun_out/r2i_tests.log; tail -1 gpurun_out/r2i_det.log; grep diagnostic gpurun_out/r2i_kernels.jsonl; tail -1 gpurun_out/r2i_kernels.jsonl
