#!/bin/bash
# prepare_kept_rows: compaction + monkey-patch + distributed tests, the default bench (e2e with
# the input pipeline preparing the targets) and the model-level step.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2bh
timeout 1500 python -m pytest tests/test_gpu_compact.py tests/test_monkey_patch.py tests/test_gpu_flce.py -m gpu -q -p no:cacheprovider > ${O}_tests.log 2>&1
tail -2 ${O}_tests.log
for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>>${O}_bench.err | tail -1 >> ${O}_bench.jsonl; done
python -c "
import json
for l in open('${O}_bench.jsonl'):
    d=json.loads(l); r=d['roofline']
    print(round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], round(r['frac'],3), {k: round(v['value']) for k,v in (d['variants'] or {}).items() if 'value' in v})"
timeout 1200 python scripts/model_step_bench.py --layers 2 --impl b200 > ${O}_model.jsonl 2>&1; tail -1 ${O}_model.jsonl
timeout 1200 python scripts/model_step_bench.py --layers 2 --impl hf > ${O}_model_hf.jsonl 2>&1; tail -1 ${O}_model_hf.jsonl
