#!/bin/bash
# chunk-size sweep: cfg2 (8192 tokens) and cfg5 at N=1 (65536 tokens), 2048 vs 4096-row chunks
cd "$GRAFT_REPO_ROOT"
for r in 1 2; do
for c in 2048 4096; do
  echo "cfg2 chunk $c: $(python bench.py --steps 20 --warmup 5 --chunk-rows $c --no-cpu-baseline --no-variants 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), d["clocks"]["sm_mhz"], d["peak_mem"]["peak_extra_minus_outputs"])')" >> gpurun_out/r2o_chunk.log
  echo "cfg5 chunk $c: $(python bench.py --config cfg5 --steps 4 --warmup 3 --chunk-rows $c --no-cpu-baseline --no-variants 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), d["clocks"]["sm_mhz"], d["peak_mem"]["peak_extra_minus_outputs"])')" >> gpurun_out/r2o_chunk.log
done; done
cat gpurun_out/r2o_chunk.log
