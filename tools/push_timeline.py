"""Print the per-op timeline of one fwd+bwd step on a one-rank peer group (push or pull) at the
configs[1] shape: which ops run on which lane and when (diagnostics of the S1/S2 overlap).

    python tools/push_timeline.py [--pull] [--n 4] [--serial]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from gpu_harness import inputs, run_gpu  # noqa: E402
from paper_2404_19429_b200 import FLAG_PEER_PUSH, FLAG_SERIAL, FLAG_TIMELINE, lancet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pull", action="store_true")
    ap.add_argument("--serial", action="store_true")
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--T", type=int, default=16384)
    ap.add_argument("--gemm-sms", type=int, default=0)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    d, f, E, k = 1024, 4096, 8, 2
    flags = FLAG_TIMELINE | (0 if a.pull else FLAG_PEER_PUSH) | (FLAG_SERIAL if a.serial else 0)
    cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=a.T, max_k=k, max_chunks=8, flags=flags,
                             gemm_sms=a.gemm_sms)
    ctx = lancet.Context(cfg, transport="peer")
    ins = inputs(a.T, d, f, E, k, beta=0.25, seed=4)
    for _ in range(4):
        run_gpu(ins, E, k, 1.25, a.n, ctx=ctx)
    tl = ctx.timeline()
    ctx.close()
    tl.sort(key=lambda o: o["start_us"])
    for o in tl:
        print(f'{o["name"]:24s} lane {o["lane"]} chunk {o["chunk"]:2d}  {o["start_us"]:9.1f} -> {o["end_us"]:9.1f}'
              f'  ({o["end_us"] - o["start_us"]:7.1f} us)')
    print(json.dumps(lancet.exposed_comm_us(tl)))
    if a.json:
        with open(a.json, "w") as fh:
            json.dump(tl, fh)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
