#!/bin/bash
# Kept X rows gathered per chunk inside the library (lk_flce_args.x_row_index): the FLCE GPU
# suites, then the bench (peak memory, speed).
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2bn
timeout 1800 python -m pytest tests/test_gpu_compact.py tests/test_gpu_flce.py tests/test_gpu_parity_headline.py tests/test_gpu_distributed.py tests/test_gpu_random.py tests/test_monkey_patch.py -m gpu -q -p no:cacheprovider > ${O}_tests.log 2>&1
tail -2 ${O}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>>${O}_bench.err | tail -1 >> ${O}_bench.jsonl; done
python -c "
import json
for l in open('${O}_bench.jsonl'):
    d=json.loads(l); r=d['roofline']; m=d['peak_mem']
    print(round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], round(r['frac'],3), round(d['ms_per_step'],3), {k: round(v,3) for k,v in r['stage_ms_per_step'].items()}, m['peak_extra_minus_outputs'], m['logits_chunk_bytes'], round(m['peak_extra_minus_outputs']/m['logits_chunk_bytes'],3))"
