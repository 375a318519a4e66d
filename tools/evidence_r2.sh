#!/bin/bash
# Round-2 evidence: full bench line (+ e2e, ep sub-record, cpu baseline) at the driver's settings
# and at the sustained defaults, the reference arm, the ncu launch list of a short bench run,
# --set full of the six GEMMs and of the SIMT kernels of one step.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2_short.json 2> gpurun_out/bench_r2_short.err
timeout 900 python bench.py > gpurun_out/bench_r2_sustained.json 2> gpurun_out/bench_r2_sustained.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r2.json 2> gpurun_out/bench_ref_r2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ep > gpurun_out/launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 18 -c 6 \
  -o gpurun_out/prof_gemm_r2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ep --flags 32 > gpurun_out/prof_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"gate_stream|slot_scan|permute|combine|k6_|dwg_|transpose" -s 27 -c 9 \
  -o gpurun_out/prof_simt_r2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ep > gpurun_out/prof_simt.log 2>&1
