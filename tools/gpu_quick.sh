#!/bin/bash
# quick GPU check: parity tests + bench (default and extra flag variants given as args)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for fl in "$@"; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --flags $fl > gpurun_out/bench_flags$fl.json 2> gpurun_out/bench_flags$fl.err
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_default2.json 2> gpurun_out/bench_default2.err
