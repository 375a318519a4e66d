#!/bin/bash
# A/B over LANCET_FLAG_* values in one session: bash tools/abf.sh rounds flagsA flagsB ...
mkdir -p gpurun_out/ab
R=$1; shift
for i in $(seq 1 $R); do
  for fl in "$@"; do
    timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --flags $fl > gpurun_out/ab/f${fl}_$i.json 2>/dev/null
  done
done
