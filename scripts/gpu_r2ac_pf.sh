#!/bin/bash
# A/B: FLCE finalize, A = row-start partial combine from L2, B = next row's partials prefetched
cd "$GRAFT_REPO_ROOT"
L=paper_2410_10989_b200/lib
for r in 1 2; do for v in A B; do
  cp $L/ab/lib$v.so $L/libliger_b200.so
  echo "$v: $(python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), d["roofline"]["stage_ms_per_step"], d["clocks"]["sm_mhz"])')" >> gpurun_out/r2ac_ab.log
  echo "$v cfg4: $(python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-variants 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), d["roofline"]["stage_ms_per_step"]["finalize"], d["clocks"]["sm_mhz"])')" >> gpurun_out/r2ac_ab.log
done; done
cp $L/ab/libB.so $L/libliger_b200.so
timeout 900 python -m pytest tests/test_gpu_flce.py tests/test_gpu_parity_headline.py tests/test_gpu_ce.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/r2ac_ab.log
timeout 600 python scripts/determinism_stage.py > gpurun_out/r2ac_det.log 2>&1
echo "differing repeats: $(grep -c '"z"' gpurun_out/r2ac_det.log)" >> gpurun_out/r2ac_ab.log
cat gpurun_out/r2ac_ab.log
