#!/bin/bash
# Functional check of bench.py's N > 1 paths on ONE GPU (never a measurement):
# GR_BENCH_ONE_GPU=1 puts both ranks on cuda:0 with the gloo backend; the
# ranks' kernels never wait on each other, only host collectives do.
#   C2/C4: one seeded batch per rank + the `strong` sub-record (one batch dealt
#          by measured cost, all-gather of the results)
#   C3:    the fused pair session, level rank ranges over the ranks
#          (all-reduce MIN of both key arrays per level)
#   C5:    clause columns over the ranks (all-reduce SUM per pick)
O=${1:-gpurun_out/onegpu}
mkdir -p $O
for c in c2 c3 c4 c5; do
  GR_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 2 --config $c \
    --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/n2_$c.json 2> $O/n2_$c.err
  echo "$c rc=$?" >> $O/rc.log
done
