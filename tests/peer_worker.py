"""Worker of tests/test_gpu_peer.py (launched by torchrun): one rank of the copy-engine peer
transport.  All ranks may share one GPU (CUDA IPC between processes of one device); the IPC
blobs are all-gathered over a gloo process group.  Writes its outputs to OUT/rank{r}.npz:
step s of `repeat` uses the inputs of seed `seed + s` (so a buffer released too early would
hand step s the rows of step s - 1), and every step's outputs are saved with suffix _s{s}.

Special modes (spec["mode"]):
  "timeout"   rank 1 never runs its step; rank 0 must come back from a bounded wait with its
              context poisoned (lancet_peer_status), and writes the message.
  "mismatch"  rank 1 creates its context with another max_tokens; import must fail on every
              rank, and each rank writes the error.
  "partitioned"  lancet_moe_forward_partitioned (every chunk gated on its own with the carried
              capacity state, per-chunk size exchange and plan) instead of lancet_moe_forward.
  "block"     the GPT-MoE block (lancet_block_*) of spec n_seq x S tokens per rank: saves out,
              h, u and the routing of each step.
"""
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


def rank_inputs(spec, r, G, step):
    Ts = spec["Ts"]
    sh = S.LayerShape(T=Ts[r], d=spec["d"], f=spec["f"], E=spec["E"], G=G, k=spec["k"], cf=1.0, n_chunks=1)
    return S.gen_rank_inputs(spec["seed"] + step, r, sh, beta=spec.get("beta", 0.5))


def main():
    spec = json.loads(os.environ["PEER_SPEC"])
    out_dir = os.environ["PEER_OUT"]
    dist.init_process_group("gloo")
    r, G = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", spec.get("device", 0))
    torch.cuda.set_device(dev)
    Ts, d, f, E, k, n = spec["Ts"], spec["d"], spec["f"], spec["E"], spec["k"], spec["n"]
    mode = spec.get("mode", "")
    bf = torch.bfloat16
    max_tokens = max(Ts) + (64 if mode == "mismatch" and r == 1 else 0)
    cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=max_tokens, max_k=k, max_chunks=8,
                             act=spec.get("act", "gelu_tanh"), flags=spec.get("flags", 0))
    if mode == "mismatch":
        try:
            lancet.Context(cfg, world=G, rank=r, device=dev.index, pg=dist.group.WORLD, transport="peer")
            msg = "created"
        except lancet.LancetError as e:
            msg = str(e)
        np.savez(os.path.join(out_dir, f"rank{r}.npz"), msg=np.array(msg))
        dist.barrier()
        dist.destroy_process_group()
        return
    if mode == "block":
        run_block(spec, r, G, dev, out_dir)
        return
    ctx = lancet.Context(cfg, world=G, rank=r, device=dev.index, pg=dist.group.WORLD, transport="peer")
    if mode == "timeout":
        ctx.set_peer_timeout_ms(spec.get("timeout_ms", 1500))
        msg = "no error"
        if r == 0:
            ins = rank_inputs(spec, r, G, 0)
            x = torch.from_numpy(ins["x"]).to(dev, bf)
            wg = torch.from_numpy(ins["wg"]).to(dev)
            w1 = torch.from_numpy(ins["w1"]).to(dev, bf)
            w2 = torch.from_numpy(ins["w2"]).to(dev, bf)
            ctx.forward(x, wg, w1, w2, k, spec["cf"], n)       # enqueues; the waits give up
            torch.cuda.synchronize()
            try:
                ctx.status()
            except lancet.LancetError as e:
                msg = str(e)
        np.savez(os.path.join(out_dir, f"rank{r}.npz"), msg=np.array(msg))
        dist.barrier()
        ctx.close()
        dist.barrier()
        dist.destroy_process_group()
        return
    res = {}
    for step in range(spec.get("repeat", 1)):
        ins = rank_inputs(spec, r, G, step)
        x = torch.from_numpy(ins["x"]).to(dev, bf)
        wg = torch.from_numpy(ins["wg"]).to(dev)
        w1 = torch.from_numpy(ins["w1"]).to(dev, bf)
        w2 = torch.from_numpy(ins["w2"]).to(dev, bf)
        dy = torch.from_numpy(ins["dy"]).to(dev, bf)
        fw = ctx.forward_partitioned if mode == "partitioned" else ctx.forward
        y, idx, slot, w = fw(x, wg, w1, w2, k, spec["cf"], n)
        dx, dwg, dw1, dw2 = ctx.backward(dy)
        torch.cuda.synchronize()
        send, recv, C = ctx.counts(n)
        one = dict(y=y.float().cpu().numpy(), idx=idx.cpu().numpy(), slot=slot.cpu().numpy(),
                   dx=dx.float().cpu().numpy(), dwg=dwg.cpu().numpy(), send=send, recv=recv, C=np.array(C))
        if dw1 is not None:
            one.update(dw1=dw1.cpu().numpy(), dw2=dw2.cpu().numpy())
        if "sample" in spec:            # large shapes: keep sampled token rows and one expert's dW
            tok = np.asarray(spec["sample"][r], dtype=np.int64)
            one["y"], one["dx"] = one["y"][tok], one["dx"][tok]
            if dw1 is not None:
                one["dw1"], one["dw2"] = one["dw1"][:1], one["dw2"][:1]
        res.update({f"{key}_s{step}": v for key, v in one.items()})
        del y, dx, dwg, dw1, dw2
    np.savez(os.path.join(out_dir, f"rank{r}.npz"), **res)
    dist.barrier()          # no rank unmaps or frees while a peer may still read its buffers
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


def run_block(spec, r, G, dev, out_dir):
    from paper_2404_19429_b200 import block as B
    bf = torch.bfloat16
    sh = S.BlockShape(n_seq=spec["n_seq"], seq_len=spec["S"], d=spec["d"], n_heads=spec["H"], f=spec["f"],
                      E=spec["E"], G=G, k=spec["k"], cf=spec["cf"], n_chunks=spec["n"])
    moe = lancet.LayerConfig(d_model=sh.d, d_ffn=sh.f, n_experts=sh.E, max_tokens=sh.T, max_k=sh.k, max_chunks=8)
    blk = B.Block(B.BlockConfig(moe, n_heads=sh.n_heads, seq_len=sh.seq_len, max_capacity_factor=sh.cf),
                  world=G, rank=r, device=dev.index, pg=dist.group.WORLD)
    res = {}
    for step in range(spec.get("repeat", 1)):
        ins = S.gen_block_rank_inputs(spec["seed"] + step, r, sh, beta=spec.get("beta", 0.5), with_dy=False)
        p = {key: torch.from_numpy(ins[key]).to(dev, torch.float32 if key in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "wg")
                                                else bf) for key in B.PARAMS}
        out = blk.forward(torch.from_numpy(ins["x"]).to(dev, bf), p, sh.k, sh.cf, sh.n_chunks)
        torch.cuda.synchronize()
        _, _, C = blk.moe.counts()
        res.update({f"out_s{step}": out.float().cpu().numpy(), f"u_s{step}": blk.debug("u", sh.T).float().numpy(),
                    f"h_s{step}": blk.debug("h", sh.T).float().numpy(), f"idx_s{step}": blk.debug("idx", sh.T).numpy(),
                    f"slot_s{step}": blk.debug("slot", sh.T).numpy(), f"C_s{step}": np.array(C)})
    np.savez(os.path.join(out_dir, f"rank{r}.npz"), **res)
    dist.barrier()
    blk.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
