#!/bin/bash
# Final bench lines on the final tree: the driver's default command, the reference arm, cfg4 /
# cfg5 / vocab-parallel at N=1, the bandwidth kernels.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2bz
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > ${O}_bench_default.jsonl 2> ${O}_bench_default.err
python bench.py --impl reference > ${O}_bench_reference.jsonl 2> ${O}_bench_reference.err
python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline > ${O}_bench_cfg4.jsonl 2>>${O}_bench.err
python bench.py --config cfg5 --steps 6 --warmup 3 --no-cpu-baseline --no-variants > ${O}_bench_cfg5.jsonl 2>>${O}_bench.err
python bench.py --mode vocab --steps 20 --warmup 3 --no-cpu-baseline --no-variants > ${O}_bench_vocab.jsonl 2>>${O}_bench.err
python bench_kernels.py > ${O}_kernels.jsonl 2>>${O}_bench.err
python -c "
import json
for f in ['default','cfg4','cfg5','vocab']:
    l=[x for x in open('${O}_bench_'+f+'.jsonl') if x.startswith('{')][-1]; d=json.loads(l); r=d['roofline']
    print(f, round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], round(r['frac'],3), d['config']['chunk_rows'], d['config']['num_chunks'], {k: round(v,3) for k,v in r['stage_ms_per_step'].items()}, {k: round(v['value']) for k,v in (d['variants'] or {}).items() if 'value' in v}, d['peak_mem']['peak_extra_minus_outputs'])
"
