#!/bin/bash
# tests + timeline-overhead A/B + bench (serial backward)
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for i in 1 2; do
  timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --flags 32 > gpurun_out/ab/tl_on_$i.json 2>/dev/null
  timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --flags 32 --no-timeline > gpurun_out/ab/tl_off_$i.json 2>/dev/null
  timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab/side_$i.json 2>/dev/null
done
