#!/bin/bash
# Peer-memory grad_w all-reduce: kernel tests (2 and 3 ranks on cuda:0 over IPC), the
# token-sharded FLCE with comm="peer", and the 2-rank shared-GPU bench path (not a bench value).
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2aw
timeout 600 python -m pytest tests/test_gpu_peer.py -m gpu -q -x -p no:cacheprovider > ${O}_peer.log 2>&1
tail -3 ${O}_peer.log
timeout 900 python -m pytest tests/test_gpu_distributed.py -m gpu -q -p no:cacheprovider > ${O}_dist.log 2>&1
tail -3 ${O}_dist.log
LK_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --bt 2048 --comm peer \
  --no-cpu-baseline --no-variants > ${O}_share_bench.log 2>&1
tail -c 600 ${O}_share_bench.log
