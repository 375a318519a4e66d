#!/bin/bash
mkdir -p gpurun_out/k6
timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"k6_stream|dwg_stream|dwg_reduce|gate_bwd_fused" -s 3 -c 6 --csv \
    --log-file gpurun_out/k6/t.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ep > /dev/null 2>&1
timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"k6_stream|dwg_stream|dwg_reduce|gate_bwd_fused" -s 3 -c 6 --csv \
    --log-file gpurun_out/k6/t_fused.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ep --flags 32 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_multirank.py -x -q > gpurun_out/k6/tests.log 2>&1; echo rc=$? >> gpurun_out/k6/tests.log
