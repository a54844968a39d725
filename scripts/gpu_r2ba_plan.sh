#!/bin/bash
# Balanced 3-chunk plan + kept-row skipping: full GPU suite, smoke, bench x2 (cfg2) + cfg4 + cfg5.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2ba
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_gputests.log 2>&1
tail -3 ${O}_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; tail -2 ${O}_smoke.log
for r in 1 2; do
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>>${O}_bench.err | tail -1 >> ${O}_bench.jsonl
done
python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-variants 2>>${O}_bench.err | tail -1 >> ${O}_bench.jsonl
python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-variants 2>>${O}_bench.err | tail -1 >> ${O}_bench.jsonl
python -c "
import json
for l in open('${O}_bench.jsonl'):
    d=json.loads(l); r=d['roofline']
    print(d['config']['workload'][:20], round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], round(r['frac'],3), d['config']['chunk_rows'], d['config']['num_chunks'], {k: round(v,3) for k,v in r['stage_ms_per_step'].items()}, {k: round(v['value']) for k,v in (d['variants'] or {}).items() if 'value' in v})"
