#!/bin/bash
# compute-sanitizer passes over small GPU tests (memcheck + racecheck + synccheck)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s3j
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
SEL_ROW='test_rmsnorm_fp32_vs_reference_golden or test_layernorm_fp32_vs_reference_golden or test_glu_fp32_vs_reference_golden or test_rope_fp32_vs_reference_golden or test_empty_inputs_all_ops'
SEL_CE='test_ce_known_answers or test_ce_golden_fp32 or test_ce_inplace_and_backward_scale'
SEL_FLCE='test_fp32_small_vs_reference_golden or test_bf16_ragged_shapes_and_bias'
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> gpurun_out/${T}_san.log
  timeout -s KILL 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_ce.py tests/test_gpu_flce.py -q -p no:cacheprovider -k "$SEL_ROW or $SEL_CE or $SEL_FLCE" > gpurun_out/${T}_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_san.log
  grep -E "ERROR SUMMARY|passed|failed|Invalid|Race|hazard" gpurun_out/${T}_$tool.log | head -8 >> gpurun_out/${T}_san.log
done
cat gpurun_out/${T}_san.log
