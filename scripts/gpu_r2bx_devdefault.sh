#!/bin/bash
# Device-count kept rows as the default: full GPU suite, smoke, bench, model-level step.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2bx
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_gputests.log 2>&1
tail -1 ${O}_gputests.log; grep FAILED ${O}_gputests.log | head -5
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>>${O}_bench.err | tail -1 >> ${O}_bench.jsonl; done
python -c "
import json
for l in open('${O}_bench.jsonl'):
    d=json.loads(l); r=d['roofline']; m=d['peak_mem']
    print(round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], round(r['frac'],3), d['config']['chunk_rows'], d['config']['num_chunks'], {k: round(v,3) for k,v in r['stage_ms_per_step'].items()}, round(d['ms_per_step'],3), m['peak_extra_minus_outputs'], {k: round(v['value']) for k,v in (d['variants'] or {}).items() if 'value' in v})"
timeout 1200 python scripts/model_step_bench.py --layers 2 > ${O}_model.jsonl 2>&1; grep impl ${O}_model.jsonl | grep -v summary
