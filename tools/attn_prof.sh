#!/bin/bash
O=gpurun_out/attn; mkdir -p $O
timeout 900 ncu --set full --clock-control none -k regex:"attn_" -c 6 -o $O/prof -f \
  python bench.py --only-block --steps 2 --warmup 1 > $O/log 2>&1
