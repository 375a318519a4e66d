#!/bin/bash
O=gpurun_out/final; mkdir -p $O
for N in 4 8; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2964$N \
    bench.py --gpus $N --steps 5 --warmup 3 --same-device --no-block > $O/bench_n${N}_same.json 2> $O/bench_n${N}_same.err; echo rc=$? >> $O/bench_n${N}_same.err
done
