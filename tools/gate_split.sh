#!/bin/bash
O=gpurun_out/gsplit; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_bpr.py tests/test_gpu_block.py -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for e in 32 64; do
  for sp in 0 1; do
    LANCET_GATE_NO_SPLIT=$sp timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"gate_" -s 3 -c 4 --csv \
      --log-file $O/e${e}_nosplit$sp.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ep --no-block --experts $e > /dev/null 2>&1
  done
done
for sp in 0 1; do
  LANCET_GATE_NO_SPLIT=$sp timeout 600 python bench.py --only-block --steps 10 --warmup 3 > $O/block_nosplit$sp.json 2>/dev/null
done
