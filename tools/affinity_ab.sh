#!/bin/bash
O=gpurun_out/aff; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1; lscpu > $O/lscpu.txt 2>&1; numactl -H > $O/numa.txt 2>&1
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-block --no-ep > $O/aff_$i.json 2>$O/aff_$i.err
  LANCET_BENCH_NO_AFFINITY=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-block --no-ep > $O/noaff_$i.json 2>/dev/null
done
