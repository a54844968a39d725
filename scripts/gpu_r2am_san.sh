#!/bin/bash
# compute-sanitizer over the piece-addressed fp32 GEMM path (new load modes 3-5) and grad_w slices
cd "$GRAFT_REPO_ROOT"
SEL='test_fp32_split_path_tiny_and_ragged_shapes or test_fp32_grad_w_slices_with_events_bitwise or test_fp32_small_vs_reference_golden or test_fp32_split_tensor_core_path_vs_oracle_and_simt'
for tool in memcheck synccheck racecheck; do
  echo "== $tool" >> gpurun_out/r2am_san.log
  timeout -s KILL 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 10 python -m pytest tests/test_gpu_flce.py tests/test_gpu_parity_headline.py -q -p no:cacheprovider -k "$SEL" > gpurun_out/r2am_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/r2am_san.log
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r2am_$tool.log | tail -2 >> gpurun_out/r2am_san.log
  grep "Race reported" -A2 gpurun_out/r2am_$tool.log | grep -v "gemm_sm100_2cta.cuh:1[56][0-9]" | grep "in .*cu.*:[0-9]" | head -3 >> gpurun_out/r2am_san.log
done
cat gpurun_out/r2am_san.log
