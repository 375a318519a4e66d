#!/bin/bash
O=gpurun_out/final; mkdir -p $O
timeout 600 python bench.py --steps 20 --warmup 5 --no-block > $O/bench_n1_auto.json 2> $O/bench_n1_auto.err; echo rc=$? >> $O/bench_n1_auto.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 \
  bench.py --gpus 2 --steps 5 --warmup 3 --same-device --no-block > $O/bench_n2_auto.json 2> $O/bench_n2_auto.err; echo rc=$? >> $O/bench_n2_auto.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_auto.json 2> $O/bench_ref_auto.err
