#!/bin/bash
# ncu --set full of the six tcgen05 GEMM launches of one step (after 3 warm-up steps)
mkdir -p gpurun_out
FL=${FL:-32}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 18 -c 6 \
  -o gpurun_out/prof_gemm -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --flags $FL > gpurun_out/prof_gemm.log 2>&1
