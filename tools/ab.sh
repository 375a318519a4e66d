#!/bin/bash
# A/B: bench ablib/libA.so (variant A) and the in-tree library (B) alternately in one session
# usage: FL=<flags> bash tools/ab.sh [rounds]
mkdir -p gpurun_out/ab
FL=${FL:-0}
R=${1:-3}
for i in $(seq 1 $R); do
  LANCET_LIB=$PWD/ablib/libA.so timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --flags $FL > gpurun_out/ab/A$i.json 2>/dev/null
  timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --flags $FL > gpurun_out/ab/B$i.json 2>/dev/null
done
