"""Lancet's ablation (dW scheduling only / pipelining only / both) on the
expert-parallel path of this implementation.

    python tools/ablation.py [--transport nccl|peer] [--chunks 4] > gpurun_out/ablation.json

Runs bench.py on the expert-parallel path (one GPU: FORCE_EP over NCCL, or the peer transport)
in four schedules:
  serial      LANCET_FLAG_SERIAL: one stream, chunks merged, dW after the exchanges
  dw_only     n = 1 with the dW GEMMs enqueued right after the dX GEMMs (they overlap the
              second backward exchange)
  pipe_only   n chunks, LANCET_FLAG_NO_DW_OVERLAP (dW after all exchanges)
  both        n chunks + dW scheduling (the default)
and prints step time and exposed all-to-all for each.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FLAG_SERIAL, FLAG_NO_DW_OVERLAP, FLAG_FORCE_EP = 4, 16, 512

ap = argparse.ArgumentParser()
ap.add_argument("--transport", choices=["nccl", "peer"], default="nccl")
ap.add_argument("--chunks", type=int, default=4)
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
base = FLAG_FORCE_EP if a.transport == "nccl" else 0
runs = {"serial": (base | FLAG_SERIAL, a.chunks), "dw_only": (base, 1),
        "pipe_only": (base | FLAG_NO_DW_OVERLAP, a.chunks), "both": (base, a.chunks)}
out = {"transport": a.transport, "chunks": a.chunks, "results": {}}
for name, (flags, n) in runs.items():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", str(a.steps), "--warmup", "4",
           "--no-e2e", "--no-cpu-baseline", "--flags", str(flags), "--chunks", str(n),
           "--transport", a.transport]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    d = json.loads(r.stdout.strip().splitlines()[-1])
    out["results"][name] = {"ms_per_step": d["ms_per_step"], "tokens_per_s": d["value"],
                            "exposed_a2a_ms": d["exposed_a2a_ms"], "a2a_ms_on_comm_lane": d["a2a_ms_on_comm_lane"]}
print(json.dumps(out, indent=1))
