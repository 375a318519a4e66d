"""Helpers shared by the -m gpu tests: run the CUDA path through the C-ABI binding and the
oracle on the same seeded inputs, and compare them.

Tolerances: routing (logits bitwise under R1, idx, slot, counts)
bit-exact; floating outputs normwise  max|gpu - ref| / max|ref|  <= 1e-2 (bf16) and <= 1e-5
(fp32 mode), the north star's "max relative error" read as in R13."""
from __future__ import annotations

import numpy as np
import torch

import synthetic as S

TOL = {"bf16": 1e-2, "fp32": 1e-5}


def normwise(got, ref) -> float:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.max(np.abs(ref))
    num = np.max(np.abs(got - ref)) if got.size else 0.0
    return float(num / den) if den > 0 else float(num)


def to_dev(a, dtype):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to(device="cuda", dtype=dtype)


def inputs(T, d, f, E, k, beta=0.5, dtype="bf16", seed=0, G=1, rank=0):
    sh = S.LayerShape(T=T, d=d, f=f, E=E, G=G, k=k, cf=1.0, n_chunks=1)
    return S.gen_rank_inputs(seed, rank, sh, beta=beta, dtype=dtype)


def run_gpu(ins, E, k, cf, n, dtype="bf16", act="gelu_tanh", flags=0, backward=True,
            max_tokens=None, ctx=None, transport="nccl"):
    from paper_2404_19429_b200 import lancet
    T, d = ins["x"].shape
    f = ins["w1"].shape[1]
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    own = ctx is None
    if own:
        cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=max_tokens or T,
                                 max_k=k, max_chunks=8, dtype=dtype, act=act, flags=flags)
        ctx = lancet.Context(cfg, transport=transport)
    x = to_dev(ins["x"], tdt)
    wg = to_dev(ins["wg"], torch.float32)
    w1 = to_dev(ins["w1"], tdt)
    w2 = to_dev(ins["w2"], tdt)
    y, idx, slot, w = ctx.forward(x, wg, w1, w2, k, cf, n)
    out = {}
    if backward:
        dy = to_dev(ins["dy"], tdt)
        dx, dwg, dw1, dw2 = ctx.backward(dy)
    torch.cuda.synchronize()
    out.update(y=y.float().cpu().numpy(), idx=idx.cpu().numpy(), slot=slot.cpu().numpy(),
               w=w.cpu().numpy(), logits=ctx.logits(T))
    send, recv, C = ctx.counts(n)
    out.update(send=send, recv=recv, C=C)
    if backward:
        out.update(dx=dx.float().cpu().numpy(), dwg=dwg.cpu().numpy())
        if dw1 is not None:
            out.update(dw1=dw1.cpu().numpy(), dw2=dw2.cpu().numpy())
    out["launches"] = ctx.launch_counts()
    if own:
        ctx.close()
    return out


def run_oracle(ins, k, cf, n, act="gelu_tanh", renorm=False, backward=True, token_subset=None,
               gate="switch", seed=0):
    from oracle import moe
    fwd = moe.forward([ins["x"]], ins["wg"], [ins["w1"]], [ins["w2"]], k, cf, n, act=act,
                      renormalize=renorm, token_subset=token_subset, gate=gate, seed=seed)
    out = dict(fwd=fwd, y=fwd.y[0], rt=fwd.routing[0])
    if backward:
        b = moe.backward(fwd, [ins["x"]], ins["wg"], [ins["w1"]], [ins["w2"]], [ins["dy"]],
                         act=act, renormalize=renorm)
        out.update(dx=b["dx"][0], dwg=b["dwg"][0])
        if "dw1" in b:
            out.update(dw1=b["dw1"][0], dw2=b["dw2"][0])
    return out


def assert_routing_exact(g, o):
    rt = o["rt"]
    assert np.array_equal(g["logits"].view(np.uint32), rt.logits.view(np.uint32)), "logits differ"
    assert np.array_equal(g["idx"], rt.idx), "expert_idx differs"
    assert np.array_equal(g["slot"], rt.slot), "slot differs"
    assert g["C"] == rt.C
    assert np.array_equal(g["send"], rt.counts), "chunk counts differ"
    assert np.allclose(g["w"], rt.w, rtol=2e-6, atol=1e-7), "combine weights differ"
