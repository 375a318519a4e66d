#!/bin/bash
# ncu: launch list of a short bench run + --set full of the SIMT kernels of one step
mkdir -p gpurun_out
FL=${1:-32}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --flags $FL > gpurun_out/launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gate_topk|slot_scan|k6_gather|dwg_partial|dwg_reduce|combine|permute" -s 21 -c 7 \
  -o gpurun_out/prof_simt -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --flags $FL > gpurun_out/prof_simt.log 2>&1
