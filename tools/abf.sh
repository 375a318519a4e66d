#!/bin/bash
# A/B over LANCET_FLAG_* values in one session: [BENCH_ARGS="..."] bash tools/abf.sh rounds flagsA flagsB ...
mkdir -p gpurun_out/ab
R=$1; shift
TAG=${TAG:-}
for i in $(seq 1 $R); do
  for fl in "$@"; do
    timeout 300 python bench.py --steps ${STEPS:-200} --warmup ${WARMUP:-100} --no-cpu-baseline --no-e2e --flags $fl $BENCH_ARGS > gpurun_out/ab/${TAG}f${fl}_$i.json 2>/dev/null
  done
done
