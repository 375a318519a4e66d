#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) on tiny configurations of every path:
# world 1, G = 2 simulated ranks (local group), one-rank peer group push / pull, and 2 processes
# over the peer transport in push mode.  Logs under gpurun_out/sanitizer/.
mkdir -p gpurun_out/sanitizer
export PYTHONFAULTHANDLER=1
for tool in memcheck racecheck synccheck; do
  for mode in world1 local2 peer1push peer1pull; do
    timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python tools/sanitize_case.py $mode > gpurun_out/sanitizer/${tool}_${mode}.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitizer/${tool}_${mode}.log
  done
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29611 \
    tools/sanitize_case.py peer2push > gpurun_out/sanitizer/${tool}_peer2push.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer/${tool}_peer2push.log
done
