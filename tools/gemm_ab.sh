#!/bin/bash
# GEMM epilogue A/B: layer parity tests on the new build, then alternate bench runs new/old,
# then an ncu --set full of the six GEMMs of one step (new build)
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_block.py -x -q > gpurun_out/gemm_tests.log 2>&1; echo rc=$? >> gpurun_out/gemm_tests.log
for i in 1 2 3; do
  timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-ep > gpurun_out/ab/new_$i.json 2>/dev/null
  LANCET_LIB=$PWD/ablib/lib_old.so timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-ep > gpurun_out/ab/old_$i.json 2>/dev/null
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 18 -c 6 \
  -o gpurun_out/prof_gemm_new -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ep --flags 32 > gpurun_out/prof_gemm.log 2>&1
