#!/bin/bash
# end-of-round checks: the whole GPU suite, memcheck / racecheck / synccheck of the round-2
# session-4 kernels, a layer-only ncu launch list
O=gpurun_out/final
mkdir -p $O gpurun_out/sanitizer
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
for tool in memcheck racecheck synccheck; do
  for mode in world1big world1big_fused; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $mode > gpurun_out/sanitizer/${tool}_${mode}.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitizer/${tool}_${mode}.log
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_layer.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ep --no-block > $O/launch_run_layer.log 2>&1
