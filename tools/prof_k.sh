#!/bin/bash
# ncu --set full of one launch of each kernel matching the regexes given (after 3 warm-up steps)
mkdir -p gpurun_out
FL=${FL:-32}
for k in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 \
    -o gpurun_out/prof_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --flags $FL > gpurun_out/prof_$k.log 2>&1
done
