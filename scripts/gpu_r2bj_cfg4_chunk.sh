#!/bin/bash
# cfg4 (Gemma-2 head, V=256000): 4 chunks of 2048 (1 GiB buffer cap) vs 3 chunks of 2560, interleaved.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2bj
for r in 1 2 3; do for c in 0 2560; do
  echo "chunk=$c $(python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-variants --chunk-rows $c 2>/dev/null | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["config"]["chunk_rows"], d["config"]["num_chunks"], {k: round(v,3) for k,v in d["roofline"]["stage_ms_per_step"].items()}, d["clocks"]["sm_mhz"], d["peak_mem"]["peak_extra_minus_outputs"])')" >> ${O}.log
done; done
cat ${O}.log
