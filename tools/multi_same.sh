#!/bin/bash
# N > 1 bench code path on one GPU (processes sharing GPU 0, peer transport): the JSON line,
# max-over-ranks timing, transport arms; not a scaling measurement
O=gpurun_out/final
mkdir -p $O
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 \
  bench.py --gpus 2 --steps 5 --warmup 3 --same-device --no-block > $O/bench_n2_same.json 2> $O/bench_n2_same.err; echo rc=$? >> $O/bench_n2_same.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29634 \
  bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $O/bench_ref_n2.json 2> $O/bench_ref_n2.err; echo rc=$? >> $O/bench_ref_n2.err
