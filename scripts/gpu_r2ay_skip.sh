#!/bin/bash
# Ignored-row skipping: compaction kernels + FLCE parity, the FLCE suites, then the bench.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2ay
timeout 1500 python -m pytest tests/test_gpu_compact.py tests/test_gpu_flce.py tests/test_gpu_parity_headline.py \
  tests/test_gpu_random.py tests/test_monkey_patch.py -m gpu -q -p no:cacheprovider > ${O}_tests.log 2>&1
tail -3 ${O}_tests.log
for r in 1 2; do
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>${O}_bench.err | tail -1 >> ${O}_bench.jsonl
done
python -c "
import json
for l in open('${O}_bench.jsonl'):
    d=json.loads(l); r=d['roofline']
    print(round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], round(r['frac'],3), {k: round(v,3) for k,v in r['stage_ms_per_step'].items()}, {k: round(v['value']) for k,v in d['variants'].items() if 'value' in v})"
