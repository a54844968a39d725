#!/bin/bash
# multi-rank code paths of bench.py on one GPU (gloo, ranks share cuda:0): correctness of the
# torchrun / token-sharded overlap / vocab-parallel plumbing, not performance
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=s3e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for M in token vocab; do
  for N in 2 4; do
    echo "== $M N=$N" >> gpurun_out/${T}_runs.log
    LK_BENCH_SHARE_GPU=1 timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --steps 3 --warmup 3 --mode $M --no-cpu-baseline > gpurun_out/${T}_${M}_${N}.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_runs.log
    tail -c 400 gpurun_out/${T}_${M}_${N}.log >> gpurun_out/${T}_runs.log; echo >> gpurun_out/${T}_runs.log
  done
done
cat gpurun_out/${T}_runs.log
