#!/bin/bash
# isolated (ncu, serialised) durations of the six GEMM launches of one step for the in-tree
# library and each ablib/lib_<name>.so variant given
mkdir -p gpurun_out/var
for v in base "$@"; do
  if [ "$v" = base ]; then L=""; else L="LANCET_LIB=$PWD/ablib/lib_$v.so"; fi
  for r in 1 2; do
    env $L timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc_gemm -s 18 -c 6 --csv \
      --log-file gpurun_out/var/${v}_$r.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ep > /dev/null 2>&1
  done
done
