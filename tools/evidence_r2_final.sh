#!/bin/bash
# Round-2 final evidence (same commands as evidence_r2.sh, current code): bench line at the
# driver's settings and at the sustained defaults, the reference arm, the ncu launch list of a
# short run, --set full of the six GEMMs and of the SIMT kernels of one step.
O=gpurun_out/final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_short.json 2> $O/bench_short.err
timeout 900 python bench.py > $O/bench_sustained.json 2> $O/bench_sustained.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ep > $O/launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 18 -c 6 \
  -o $O/prof_gemm -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ep --flags 32 > $O/prof_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"gate_stream|slot_scan|permute|combine|k6_|dwg_|transpose" -s 27 -c 9 \
  -o $O/prof_simt -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ep > $O/prof_simt.log 2>&1
