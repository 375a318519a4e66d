#!/bin/bash
# A/B/n: bench the in-tree library ("base") and each ablib/lib_<name>.so given, alternately
# usage: FL=<flags> bash tools/abn.sh rounds name1 name2 ...
mkdir -p gpurun_out/ab
FL=${FL:-0}
R=$1; shift
for i in $(seq 1 $R); do
  timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --flags $FL > gpurun_out/ab/base_$i.json 2>/dev/null
  for v in "$@"; do
    LANCET_LIB=$PWD/ablib/lib_$v.so timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --flags $FL > gpurun_out/ab/${v}_$i.json 2>/dev/null
  done
done
