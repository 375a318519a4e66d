"""One tiny fwd+bwd (two steps, different inputs) of a path, for compute-sanitizer runs
(tools/sanitize.sh): world1 | local2 | peer1push | peer1pull | peer2push (under torchrun)."""
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
