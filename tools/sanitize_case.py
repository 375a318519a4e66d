"""One tiny fwd+bwd (two steps, different inputs) of a path, for compute-sanitizer runs
(tools/sanitize.sh): world1 | local2 | peer1push | peer1pull | peer2push (under torchrun) |
partitioned (lancet_moe_forward_partitioned + backward) | block (block forward + backward, and a
two-block stack forward)."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import synthetic as S  # noqa: E402
from paper_2404_19429_b200 import FLAG_PEER_PUSH, lancet  # noqa: E402

T, d, f, E, k, n = 300, 128, 256, 4, 2, 2


def run(ctx, rank, G, steps=2):
    dev = torch.device("cuda", 0)
    bf = torch.bfloat16
    for s in range(steps):
        sh = S.LayerShape(T=T, d=d, f=f, E=E, G=G, k=k, cf=1.0, n_chunks=n)
        ins = S.gen_rank_inputs(5 + s, rank, sh, beta=0.5)
        x = torch.from_numpy(ins["x"]).to(dev, bf)
        wg = torch.from_numpy(ins["wg"]).to(dev)
        w1 = torch.from_numpy(ins["w1"]).to(dev, bf)
        w2 = torch.from_numpy(ins["w2"]).to(dev, bf)
        dy = torch.from_numpy(ins["dy"]).to(dev, bf)
        ctx.forward(x, wg, w1, w2, k, 1.0, n)
        ctx.backward(dy)
        torch.cuda.synchronize()


def main():
    mode = sys.argv[1]
    mk = lambda fl=0: lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k, max_chunks=4,  # noqa
                                         flags=fl)
    if mode == "world1":
        c = lancet.Context(mk())
        run(c, 0, 1)
        c.close()
    elif mode in ("peer1push", "peer1pull"):
        c = lancet.Context(mk(FLAG_PEER_PUSH if mode == "peer1push" else 0), transport="peer")
        run(c, 0, 1)
        c.close()
    elif mode == "local2":
        g = lancet.LocalGroup(2)
        errs = []

        def w(r):
            try:
                torch.cuda.set_device(0)
                c = lancet.Context(mk(), world=2, rank=r, device=0, local_group=g)
                with torch.cuda.stream(torch.cuda.Stream()):
                    run(c, r, 2)
                c.close()
            except Exception as e:  # noqa: BLE001
                errs.append(e)
        th = [threading.Thread(target=w, args=(r,)) for r in range(2)]
        [t.start() for t in th]
        [t.join() for t in th]
        g.close()
        assert not errs, errs
    elif mode == "partitioned":
        c = lancet.Context(mk(FLAG_PEER_PUSH), transport="peer")
        dev = torch.device("cuda", 0)
        for s_ in range(2):
            sh = S.LayerShape(T=T, d=d, f=f, E=E, G=1, k=k, cf=1.0, n_chunks=n)
            ins = S.gen_rank_inputs(5 + s_, 0, sh, beta=0.5)
            x, wg, w1, w2, dy = (torch.from_numpy(ins[key]).to(dev, torch.float32 if key == "wg" else torch.bfloat16)
                                 for key in ("x", "wg", "w1", "w2", "dy"))
            c.forward_partitioned(x, wg, w1, w2, k, 1.0, n)
            c.backward(dy)
            torch.cuda.synchronize()
        c.close()
    elif mode == "block":
        from paper_2404_19429_b200 import block as B
        sh = S.BlockShape(n_seq=2, seq_len=128, d=256, n_heads=2, f=256, E=4, G=1, k=2, cf=1.0, n_chunks=2)
        ins = S.gen_block_rank_inputs(9, 0, sh, beta=0.5)
        dev = torch.device("cuda", 0)
        p = {key: torch.from_numpy(ins[key]).to(dev, torch.float32 if key in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "wg")
                                                else torch.bfloat16) for key in B.PARAMS}
        moe = lancet.LayerConfig(d_model=sh.d, d_ffn=sh.f, n_experts=sh.E, max_tokens=sh.T, max_k=sh.k, max_chunks=4)
        blks = [B.Block(B.BlockConfig(moe, n_heads=sh.n_heads, seq_len=sh.seq_len, max_capacity_factor=1.0))
                for _ in range(2)]
        x = torch.from_numpy(ins["x"]).to(dev, torch.bfloat16)
        out = blks[0].forward(x, p, sh.k, sh.cf, 2)
        blks[0].backward(torch.from_numpy(ins["dy"]).to(dev, torch.bfloat16))
        outs = B.forward_stack(blks, x, [p, p], sh.k, sh.cf, 2)
        g = blks[1].backward(outs[1])
        blks[0].backward(g["dx"])
        torch.cuda.synchronize()
        for b_ in blks:
            b_.close()
        del out
    elif mode == "peer2push":
        import torch.distributed as dist
        dist.init_process_group("gloo")
        r, G = dist.get_rank(), dist.get_world_size()
        torch.cuda.set_device(0)
        c = lancet.Context(mk(FLAG_PEER_PUSH), world=G, rank=r, device=0, pg=dist.group.WORLD, transport="peer")
        run(c, r, G)
        dist.barrier()
        c.close()
        dist.barrier()
        dist.destroy_process_group()
    print("ok", mode)


if __name__ == "__main__":
    main()
