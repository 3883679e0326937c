#!/bin/bash
# The sharded (N>1) bench path on a 1-GPU box: N ranks share cuda:0 over gloo.
OUT=gpurun_out; mkdir -p $OUT
for N in 2 4; do
COSCHED_BENCH_SHARE_GPU=1 COSCHED_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 5 --warmup 3 --no-cpu-baseline \
  > $OUT/bench_dist$N.json 2> $OUT/bench_dist$N.err
echo "N=$N rc=$?" >> $OUT/bench_dist.rc
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo "ref rc=$?" >> $OUT/bench_dist.rc
