#!/bin/bash
# compute-sanitizer over the round-2 kernel changes: chunked GLU / RoPE, CE ring release, segmented
# fp32 accumulation (split-operand FLCE), GEMM use-counter refactor
cd "$GRAFT_REPO_ROOT"
T=r2ab
SEL_ROW='test_glu_fp32_vs_reference_golden or test_glu_unaligned_views_vs_torch or test_rope_all_tokens_vs_torch or test_rope_per_batch_tables or test_empty_inputs_all_ops or test_swiglu_gate_and_down_multipliers'
SEL_CE='test_ce_known_answers or test_ce_golden_fp32'
SEL_FLCE='test_fp32_small_vs_reference_golden or test_fp32_split_tensor_core_path_vs_oracle_and_simt'
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> gpurun_out/${T}_san.log
  timeout -s KILL 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_ce.py tests/test_gpu_flce.py tests/test_gpu_parity_headline.py -q -p no:cacheprovider -k "$SEL_ROW or $SEL_CE or $SEL_FLCE" > gpurun_out/${T}_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_san.log
  grep -E "ERROR SUMMARY|passed|failed|Invalid|Race|hazard" gpurun_out/${T}_$tool.log | head -8 >> gpurun_out/${T}_san.log
done
cat gpurun_out/${T}_san.log
timeout 600 python bench.py --mode vocab --steps 20 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/r2ab_bench_vocab_n1.jsonl 2>&1
tail -c 700 gpurun_out/r2ab_bench_vocab_n1.jsonl
