#!/bin/bash
# compute-sanitizer memcheck / synccheck / racecheck on the round-2 additions: the partitioned
# MoE forward and the GPT-MoE block (forward, backward, two-block stack).  Logs under
# gpurun_out/sanitizer/.
mkdir -p gpurun_out/sanitizer
for tool in memcheck synccheck racecheck; do
  for mode in partitioned block; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $mode \
      > gpurun_out/sanitizer/${tool}_${mode}.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitizer/${tool}_${mode}.log
  done
done
