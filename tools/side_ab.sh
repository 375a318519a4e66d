#!/bin/bash
O=gpurun_out/side; mkdir -p $O
for i in 1 2 3; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-ep --no-block --no-timeline > $O/side_$i.json 2>/dev/null
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-ep --no-block --no-timeline --flags 32 > $O/fused_$i.json 2>/dev/null
done
