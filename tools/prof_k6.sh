#!/bin/bash
mkdir -p gpurun_out/k6
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k6_stream|combine_bwd|dwg_stream|permute_kernel|combine_kernel" -s 5 -c 5 \
  -o gpurun_out/k6/prof -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ep > gpurun_out/k6/log 2>&1
