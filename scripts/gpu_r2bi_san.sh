#!/bin/bash
# compute-sanitizer over the kernels added late in round 2: row compaction / gather (and the FLCE
# on kept rows), the peer-memory all-reduce (2 processes on one GPU; every child process
# sanitized), and the vectorised register dW accumulate path.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2bi
SEL='test_compact_rows_matches_numpy or test_gather_rows_every_width_and_fill or (test_flce_skip_ignored_rows_vs_full_call_and_oracle and (default or reduction or _frac)) or test_prepared_kept_rows'
for tool in memcheck synccheck racecheck; do
  echo "== $tool compact" >> ${O}_san.log
  timeout -s KILL 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 10 python -m pytest tests/test_gpu_compact.py -q -p no:cacheprovider -k "$SEL" > ${O}_compact_$tool.log 2>&1; echo "rc=$?" >> ${O}_san.log
  grep -E "ERROR SUMMARY|passed|failed" ${O}_compact_$tool.log | tail -2 >> ${O}_san.log
  grep "Race reported" -A2 ${O}_compact_$tool.log | grep -v "gemm_sm100_2cta.cuh:1[5-9][0-9]" | grep "in .*cu.*:[0-9]" | head -3 >> ${O}_san.log
done
for tool in memcheck synccheck; do
  echo "== $tool peer" >> ${O}_san.log
  timeout -s KILL 900 compute-sanitizer --tool $tool --target-processes all --error-exitcode 9 --print-limit 10 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider -k "bitwise and 2" > ${O}_peer_$tool.log 2>&1; echo "rc=$?" >> ${O}_san.log
  grep -E "ERROR SUMMARY|passed|failed" ${O}_peer_$tool.log | tail -3 >> ${O}_san.log
done
echo "== memcheck accum16 register path" >> ${O}_san.log
timeout -s KILL 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 10 python -m pytest tests/test_gpu_flce.py -q -p no:cacheprovider -k "test_weight_dtype_accumulation_paths_vs_oracle" > ${O}_acc16.log 2>&1; echo "rc=$?" >> ${O}_san.log
grep -E "ERROR SUMMARY|passed|failed" ${O}_acc16.log | tail -2 >> ${O}_san.log
cat ${O}_san.log
