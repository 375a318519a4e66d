"""Single-GPU shape sweep (SURVEY §8(d) config 5 at N=1): tokens/GPU x experts x chunks.

    python tools/sweep.py [--quick] > gpurun_out/sweep.jsonl

Each line is bench.py's JSON for one shape (no e2e / cpu baseline), so per-op times and the
GEMM roofline come along.  Multi-GPU points need torchrun on a multi-GPU node (bench.py --gpus N).
"""
import argparse
import json
import subprocess
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true")
a = ap.parse_args()
shapes = []
for E in (8, 16, 32, 64):
    for T in (4096, 16384, 65536):
        shapes.append((T, E, 0))
if a.quick:
    shapes = shapes[:3]
for T, E, n in shapes:
    cmd = [sys.executable, "bench.py", "--steps", "20", "--warmup", "4", "--no-e2e", "--no-cpu-baseline",
           "--no-ep", "--no-block", "--tokens", str(T), "--experts", str(E), "--chunks", str(n)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps({"error": r.stderr[-400:]})
    d = json.loads(line)
    d["sweep"] = {"tokens_per_gpu": T, "experts": E, "n_chunks": n}
    print(json.dumps(d), flush=True)
