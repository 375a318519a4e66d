#!/bin/bash
O=gpurun_out/attn; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_block.py -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for v in new old; do
  if [ $v = old ]; then L="LANCET_LIB=$PWD/ablib/lib_ATTN2.so"; else L=""; fi
  env $L timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"attn_fwd" -c 8 --csv \
    --log-file $O/t_$v.csv python bench.py --only-block --steps 2 --warmup 1 > /dev/null 2>&1
  env $L timeout 600 python bench.py --only-block --steps 10 --warmup 3 > $O/block_$v.json 2>/dev/null
done
