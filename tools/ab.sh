#!/bin/bash
# A/B: bench the in-tree library and gpurun_out/ab/libA.so alternately in one session
mkdir -p gpurun_out/ab
for i in 1 2; do
  LANCET_LIB=$PWD/ablib/libA.so python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab/A$i.json 2>/dev/null
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab/B$i.json 2>/dev/null
done
for f in A1 B1 A2 B2; do echo $f; python profiles/show_bench.py gpurun_out/ab/$f.json | head -8; done
