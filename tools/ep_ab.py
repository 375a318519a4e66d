"""A/B of the push-mode schedules on a one-rank peer group at the configs[1] shape: ms per
fwd+bwd step (CUDA events, K steps after W warm-up) for n in {1, 2, 4, 8}, device-side GEMM
pipeline (default) vs per-chunk launches vs the serial baseline.

    python tools/ep_ab.py [--steps 30] [--warmup 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from gpu_harness import inputs, to_dev  # noqa: E402
from paper_2404_19429_b200 import FLAG_CHUNK_LAUNCHES, FLAG_PEER_PUSH, FLAG_SERIAL, lancet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--T", type=int, default=16384)
    ap.add_argument("--E", type=int, default=8)
    ap.add_argument("--ns", default="1,2,4,8")
    ap.add_argument("--rounds", type=int, default=2)
    a = ap.parse_args()
    d, f, k, E, T = 1024, 4096, 2, a.E, a.T
    ins = inputs(T, d, f, E, k, beta=0.25, seed=4)
    bf = torch.bfloat16
    x, dy = to_dev(ins["x"], bf), to_dev(ins["dy"], bf)
    wg, w1, w2 = to_dev(ins["wg"], torch.float32), to_dev(ins["w1"], bf), to_dev(ins["w2"], bf)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    dwg = torch.empty_like(wg)
    dw1, dw2 = torch.empty(w1.shape, device="cuda"), torch.empty(w2.shape, device="cuda")
    modes = {"pipelined": 0, "chunk_launches": FLAG_CHUNK_LAUNCHES, "serial": FLAG_SERIAL}
    ctxs = {m: lancet.Context(lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k, max_chunks=8,
                                                 flags=FLAG_PEER_PUSH | fl), transport="peer")
            for m, fl in modes.items()}
    res = {}
    for rnd in range(a.rounds):
        for n in [int(v) for v in a.ns.split(",")]:
            for m, ctx in ctxs.items():
                def step():
                    ctx.forward(x, wg, w1, w2, k, 1.25, n, y=y, routing=False)
                    ctx.backward(dy, dx=dx, dwg=dwg, dw1=dw1, dw2=dw2)
                for _ in range(a.warmup):
                    step()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.steps):
                    step()
                e1.record()
                torch.cuda.synchronize()
                res.setdefault(f"{m} n={n}", []).append(e0.elapsed_time(e1) / a.steps)
    for key, v in res.items():
        print(f"{key:28s} " + " ".join(f"{t:.3f}" for t in v) + " ms")
    print(json.dumps(res))
    for c in ctxs.values():
        c.close()


if __name__ == "__main__":
    main()
