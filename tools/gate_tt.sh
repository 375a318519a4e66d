#!/bin/bash
# gate tokens-per-thread A/B: isolated ncu durations (bench step, configs[1]) at E = 8 / 16
mkdir -p gpurun_out/gtt
rm -f gpurun_out/gtt/*.csv
for tt in 1 2; do
  for e in 8 16; do
  LANCET_GATE_TT=$tt timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second -k regex:"gate_stream|gate_topk" -s 2 -c 3 --csv \
    --log-file gpurun_out/gtt/tt${tt}_e$e.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ep --experts $e > /dev/null 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_bpr.py -x -q > gpurun_out/gtt/tests.log 2>&1; echo rc=$? >> gpurun_out/gtt/tests.log
LANCET_GATE_TT=1 timeout 900 python -m pytest tests/test_gpu_layer.py -x -q -k "routing or parity" > gpurun_out/gtt/tests2.log 2>&1; echo rc=$? >> gpurun_out/gtt/tests2.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ep > gpurun_out/gtt/bench.json 2>/dev/null
