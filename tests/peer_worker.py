"""Worker of tests/test_gpu_peer.py (launched by torchrun): one rank of the copy-engine peer
transport.  All ranks may share one GPU (CUDA IPC between processes of one device); the IPC
blobs are all-gathered over a gloo process group.  Writes its outputs to OUT/rank{r}.npz."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import synthetic as S  # noqa: E402
from paper_2404_19429_b200 import lancet  # noqa: E402


def main():
    spec = json.loads(os.environ["PEER_SPEC"])
    out_dir = os.environ["PEER_OUT"]
    dist.init_process_group("gloo")
    r, G = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", spec.get("device", 0))
    torch.cuda.set_device(dev)
    Ts, d, f, E, k, n = spec["Ts"], spec["d"], spec["f"], spec["E"], spec["k"], spec["n"]
    sh = S.LayerShape(T=Ts[r], d=d, f=f, E=E, G=G, k=k, cf=1.0, n_chunks=1)
    ins = S.gen_rank_inputs(spec["seed"], r, sh, beta=spec.get("beta", 0.5))
    bf = torch.bfloat16
    x = torch.from_numpy(ins["x"]).to(dev, bf)
    wg = torch.from_numpy(ins["wg"]).to(dev)
    w1 = torch.from_numpy(ins["w1"]).to(dev, bf)
    w2 = torch.from_numpy(ins["w2"]).to(dev, bf)
    dy = torch.from_numpy(ins["dy"]).to(dev, bf)
    cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=max(Ts), max_k=k, max_chunks=8,
                             act=spec.get("act", "gelu_tanh"), flags=spec.get("flags", 0))
    ctx = lancet.Context(cfg, world=G, rank=r, device=dev.index, pg=dist.group.WORLD, transport="peer")
    for _ in range(spec.get("repeat", 1)):
        y, idx, slot, w = ctx.forward(x, wg, w1, w2, k, spec["cf"], n)
        dx, dwg, dw1, dw2 = ctx.backward(dy)
    torch.cuda.synchronize()
    send, recv, C = ctx.counts(n)
    res = dict(y=y.float().cpu().numpy(), idx=idx.cpu().numpy(), slot=slot.cpu().numpy(),
               dx=dx.float().cpu().numpy(), dwg=dwg.cpu().numpy(), send=send, recv=recv, C=np.array(C))
    if dw1 is not None:
        res.update(dw1=dw1.cpu().numpy(), dw2=dw2.cpu().numpy())
    np.savez(os.path.join(out_dir, f"rank{r}.npz"), **res)
    dist.barrier()          # no rank unmaps or frees while a peer may still read its buffers
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
