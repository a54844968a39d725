#!/bin/bash
# compute-sanitizer over the kernels changed this session: CE ring (32 KB pieces), weights+smoothing
# block CE, PDL column sums, token-major RoPE, SwiGLU gate multiplier, wide-row norms
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s4g
SEL_ROW='test_rmsnorm_fp32_vs_reference_golden or test_layernorm_fp32_vs_reference_golden or test_rope_all_tokens_vs_torch or test_swiglu_gate_and_down_multipliers or test_norms_wide_rows_vs_torch or test_empty_inputs_all_ops'
SEL_CE='test_ce_known_answers or test_ce_golden_fp32 or test_ce_class_weights'
SEL_FLCE='test_fp32_small_vs_reference_golden or test_flce_ce_weight'
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> gpurun_out/${T}_san.log
  timeout -s KILL 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_ce.py tests/test_gpu_flce.py -q -p no:cacheprovider -k "$SEL_ROW or $SEL_CE or $SEL_FLCE" > gpurun_out/${T}_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_san.log
  grep -E "ERROR SUMMARY|passed|failed|Invalid|Race|hazard" gpurun_out/${T}_$tool.log | head -8 >> gpurun_out/${T}_san.log
done
cat gpurun_out/${T}_san.log
