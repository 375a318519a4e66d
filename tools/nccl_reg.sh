#!/bin/bash
O=gpurun_out/nreg; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_multirank.py tests/test_gpu_tuner.py -x -q -s -k "nccl or force_ep or multirank or tune or layer" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for r in 1 0; do
  LANCET_NCCL_REGISTER=$r timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-ep --no-block --flags 512 > $O/bench_force_ep_reg$r.json 2> $O/bench_force_ep_reg$r.err
done
