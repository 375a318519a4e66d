"""Cross-layer dW scheduling on an L-layer stack (PAPER.md Opportunity 1, Alg. 1; R17).

    python tools/stack_dw.py [--layers 4] [--transport peer|nccl] [--chunks 1 2] > out.json

One GPU, every layer on the expert-parallel path (peer: the copy-engine transport as a one-rank
group; nccl: FORCE_EP over a one-rank communicator), BASELINE configs[1] layer shape.  For each
chunk count, three schedules of the same stack fwd+bwd:
  late   every layer's dW GEMMs after all its all-to-alls (LANCET_FLAG_NO_DW_OVERLAP): no dW
         scheduling;
  own    every layer's dW right after its own dX GEMMs (the library default: they overlap the
         layer's own dX return);
  alg1   Alg. 1 over the whole stack (lancet_stack_dw_plan) with per-op costs measured from a
         timeline of `own`: dW GEMMs may move under later layers' dO dispatch;
and reports ms per stack step (CUDA events, after warm-up) and the exposed all-to-all time over
the union of all layers' timelines.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synthetic as S  # noqa: E402
from paper_2404_19429_b200 import lancet  # noqa: E402
from paper_2404_19429_b200.stack import MoEStack, costs_from_timelines, plan_from_costs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--transport", choices=["peer", "nccl"], default="peer")
ap.add_argument("--chunks", type=int, nargs="+", default=[1, 2])
ap.add_argument("--tokens", type=int, default=16384)
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--warmup", type=int, default=40)
ap.add_argument("--rounds", type=int, default=7)
a = ap.parse_args()

L, T, d, f, E, k, cf = a.layers, a.tokens, 1024, 4096, 8, 2, 1.25
base = lancet.FLAG_FORCE_EP if a.transport == "nccl" else 0
ctxs = [lancet.Context(lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k,
                                          max_chunks=8, flags=base), transport=a.transport)
        for _ in range(L)]
stack = MoEStack(ctxs)
params, grads = [], []
for l in range(L):
    sh = S.LayerShape(T=T, d=d, f=f, E=E, G=1, k=k, cf=cf, n_chunks=1)
    ins = S.gen_rank_inputs(300 + l, 0, sh, beta=0.25)
    params.append((torch.from_numpy(ins["wg"]).cuda(), torch.from_numpy(ins["w1"]).cuda().bfloat16(),
                   torch.from_numpy(ins["w2"]).cuda().bfloat16()))
    grads.append((torch.empty_like(params[-1][0]), torch.empty(params[-1][1].shape, device="cuda"),
                  torch.empty(params[-1][2].shape, device="cuda")))
    if l == 0:
        x = torch.from_numpy(ins["x"]).cuda().bfloat16()
        dy = torch.from_numpy(ins["dy"]).cuda().bfloat16()
stream = torch.cuda.current_stream()


def set_flags(extra):
    for c in ctxs:
        c.set_flags(base | extra)


def step(n, plan):
    stack.forward(x, params, k, cf, n)
    stack.backward(dy, grads, plan=plan)


def time_once(n, plan, extra):
    set_flags(extra)
    step(n, plan)                      # the first step after a schedule switch is not timed
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        step(n, plan)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.steps


def exposure(n, plan, extra):
    # timeline pass: exposure over the union of all layers' timelines (one common base)
    set_flags(extra | lancet.FLAG_TIMELINE)
    step(n, plan)
    torch.cuda.synchronize()
    for c in ctxs:
        c.timeline_begin(stream)
    ns = 3
    for _ in range(ns):
        step(n, plan)
    torch.cuda.synchronize()
    tls = [c.timeline(cap=100000) for c in ctxs]
    set_flags(extra)
    union = [r for tl in tls for r in tl]
    ex = lancet.exposed_comm_us(union)
    bwd_a2a = [r for r in union if r["lane"] == 1 and r["name"].startswith("a2a_bwd")]
    ex_b = lancet.exposed_comm_us([r for r in union if r["lane"] != 1] + bwd_a2a)
    return dict(exposed_a2a_ms=ex["exposed_us"] / ns / 1000.0, a2a_ms=ex["comm_us"] / ns / 1000.0,
                exposed_bwd_a2a_ms=ex_b["exposed_us"] / ns / 1000.0), tls


out = {"layers": L, "transport": a.transport, "tokens_per_layer": T,
       "shape": f"d={d} f={f} E={E} top-{k} cf={cf} bf16", "steps_per_sample": a.steps,
       "rounds": a.rounds, "timing": "median over rounds of K stack fwd+bwd steps per schedule, "
       "schedules interleaved round by round after a warm-up into the power-capped regime",
       "results": {}}
for n in a.chunks:
    res = {"late": {}, "own": {}, "alg1": {}}
    res["late"].update(exposure(n, None, lancet.FLAG_NO_DW_OVERLAP)[0])
    ex_own, tls = exposure(n, None, 0)
    res["own"].update(ex_own)
    t_a2a, t_dw = costs_from_timelines(tls, n)
    hl, ha = plan_from_costs(t_a2a, t_dw)
    res["alg1"].update(exposure(n, (hl, ha), 0)[0])
    scheds = {"late": (None, lancet.FLAG_NO_DW_OVERLAP), "own": (None, 0), "alg1": ((hl, ha), 0)}
    set_flags(0)
    for _ in range(a.warmup):
        step(n, None)
    samples = {s_: [] for s_ in scheds}
    for _ in range(a.rounds):
        for name, (plan, extra) in scheds.items():
            samples[name].append(time_once(n, plan, extra))
    for name in scheds:
        ms = float(np.median(samples[name]))
        res[name].update(ms_per_step=ms, stack_tokens_per_s=T / (ms / 1000.0),
                         samples_ms=[round(v, 3) for v in samples[name]])
    res["plan"] = {"host_layer": hl.tolist(), "host_a2a": ha.tolist(),
                   "t_a2a_us": np.round(t_a2a, 1).tolist(), "t_dw_us": np.round(t_dw, 1).tolist()}
    out["results"][f"n={n}"] = res
print(json.dumps(out, indent=1))
