#!/bin/bash
# Kept-row skipping in the token-sharded and vocab-parallel modes: GPU distributed tests, the
# vocab-parallel N=1 bench, and the 2-rank shared-GPU path checks (not bench values).
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2bf
timeout 1500 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_compact.py -m gpu -q -p no:cacheprovider > ${O}_tests.log 2>&1
tail -3 ${O}_tests.log
python bench.py --mode vocab --steps 20 --warmup 3 --no-cpu-baseline > ${O}_vocab.jsonl 2>${O}_vocab.err
for mode in token vocab; do
LK_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 \
  --master-addr 127.0.0.1 --master-port 2954$([ $mode = token ] && echo 1 || echo 2) bench.py --gpus 2 --mode $mode --steps 3 --warmup 3 --bt 4096 \
  --no-cpu-baseline --no-variants > ${O}_share_$mode.log 2>&1
done
python -c "
import json
for f in ['vocab.jsonl','share_token.log','share_vocab.log']:
    ls=[x for x in open('${O}_'+f) if x.startswith('{')]
    if not ls: print(f, 'NO LINE'); continue
    d=json.loads(ls[-1]); r=d['roofline']
    print(f, round(d['value']), round(d['e2e']['value']), round(r['frac'],3), r['ignored_rows_skipped'], d['config']['chunk_rows'], {k: round(v['value']) for k,v in (d['variants'] or {}).items() if 'value' in v})"
