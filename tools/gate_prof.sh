#!/bin/bash
mkdir -p gpurun_out/gtt
for tt in 1 2; do
LANCET_GATE_TT=$tt timeout 600 ncu --set full --import-source on --clock-control none -k regex:gate_stream -s 2 -c 1 \
  -o gpurun_out/gtt/prof_tt$tt -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ep > /dev/null 2>&1
done
