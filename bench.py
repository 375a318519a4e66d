#!/usr/bin/env python
"""bench.py -- MoE layer fwd+bwd tokens/s on B200 (BASELINE.json metric), plus exposed
all-to-all ms/iter, roofline of the dominant kernel, end-to-end (host buffers) throughput and
the CPU oracle baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lancet|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1, one rank per GPU)

Workload (BASELINE.json configs[1], per GPU): GPT-MoE layer d_model=1024, ffn=4096, E=8
experts in total (E/N per GPU), top-2, capacity factor 1.25, 16384 tokens per GPU, bf16,
n_chunks=4, synthetic inputs (synthetic/, routing skew beta=0.25).  One step = forward +
backward of the layer through the C-ABI (lancet_moe_forward / lancet_moe_backward).

--impl reference times the CPU oracle (oracle/, the reference arm of this tier) on bounded
samples of the same workload, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE layer fwd+bwd tokens/s at 1/2/4/8 B200; exposed all-to-all ms/iter"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # defaults measure the sustained regime: a B200 under this load reaches its power cap
    # (sw_power_cap, ~1.2 GHz) within ~100 ms; a 5-step warm-up would time boost clocks
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--impl", choices=["lancet", "reference"], default="lancet")
    ap.add_argument("--tokens", type=int, default=16384, help="tokens per GPU")
    ap.add_argument("--d", type=int, default=1024)
    ap.add_argument("--f", type=int, default=4096)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--cf", type=float, default=1.25)
    ap.add_argument("--chunks", type=int, default=0,
                    help="chunk count n of the expert-parallel pipeline; 0 = auto: at N > 1 the "
                         "fastest of n = 1, 2, 4, 8 in a short probe on this run's ranks (the "
                         "paper picks n by search, P:L411-L414); at N = 1 the single-GPU path has "
                         "no exchange to pipeline and runs unchunked")
    ap.add_argument("--beta", type=float, default=0.25)
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--flags", type=int, default=0, help="extra LANCET_FLAG_* bits")
    ap.add_argument("--gate", choices=["switch", "bpr", "random"], default="switch",
                    help="token-major top-k (Switch/GShard-style), Batch Prioritized Routing "
                         "(PAPER.md L270; LANCET_FLAG_GATE_BPR) or the Random gate (L271; "
                         "LANCET_FLAG_GATE_RANDOM, seed 0)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--transport", choices=["auto", "nccl", "peer"], default="auto",
                    help="world > 1: NCCL grouped send/recv, copy-engine pulls over CUDA IPC, or "
                         "auto (peer if every rank can set it up, else NCCL)")
    ap.add_argument("--no-push", action="store_true",
                    help="peer transport: pull the dispatch rows with the copy engines instead of "
                         "pushing them from the permute kernel (LANCET_FLAG_PEER_PUSH)")
    ap.add_argument("--same-device", action="store_true",
                    help="all ranks on GPU 0 (peer transport, gloo process group): a multi-process "
                         "test of the exchange machinery on one GPU, not a scaling measurement")
    ap.add_argument("--no-timeline", action="store_true",
                    help="no per-op events in the timed region (A/B of their overhead)")
    ap.add_argument("--no-ep", action="store_true",
                    help="N = 1: skip the 'ep' sub-record (the expert-parallel chunk pipeline over a "
                         "one-rank peer group, with its exposure and no-comm differential)")
    ap.add_argument("--no-block", action="store_true",
                    help="skip the 'block' sub-record (BASELINE configs[3]: the GPT-MoE block forward "
                         "with the pre-MoE partition, NEXT-1)")
    ap.add_argument("--only-block", action="store_true",
                    help="measure and print only the 'block' record")
    ap.add_argument("--no-arms", action="store_true",
                    help="N > 1: skip the per-transport arms (push / pull / NCCL on one definition)")
    a = ap.parse_args()
    a.warmup = max(a.warmup, 3)
    a.chunks_req = a.chunks
    if a.chunks <= 0:
        a.chunks = 4           # provisional (shapes, oracle calls: results do not depend on n)
    if a.same_device:
        a.transport = "peer"
    return a


def _nlabel(a):
    return "auto" if getattr(a, "chunks_req", a.chunks) <= 0 else a.chunks


def workload(a, world):
    return {
        "workload": f"GPT-MoE layer fwd+bwd: d_model={a.d} ffn={a.f} experts={a.experts} "
                    f"({a.experts // world}/GPU) top-{a.k} cf={a.cf} {a.tokens} tokens/GPU "
                    f"n_chunks={_nlabel(a)} bf16" + ("" if a.gate == "switch" else f" gate={a.gate}"),
        "tokens_per_gpu": a.tokens, "d_model": a.d, "d_ffn": a.f, "experts": a.experts,
        "top_k": a.k, "capacity_factor": a.cf, "n_chunks": _nlabel(a), "routing_skew_beta": a.beta,
        "gate": a.gate,
        "parallelism": f"ep{world}" + (f" ({getattr(a, 'transport_used', a.transport)}"
                                       + (" push" if getattr(a, "transport_used", "") == "peer" and not a.no_push else "")
                                       + " all-to-all)"
                                       if world > 1 or a.transport == "peer" else "")
                       + (" all ranks on one GPU" if getattr(a, "same_device", False) else ""),
        "global_batch_tokens": a.tokens * world,
        "l2": "inputs larger than L2: per-step working set >= 1.4 GiB vs 126 MB L2 (no flush)",
    }


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return dict(hbm=j["hbm_gbs"], bf16=j["bf16_tflops"], bf16_sus=j.get("bf16_tflops_sustained", j["bf16_tflops"]),
                    src="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback (B200_PROFILING.md)")


def gemm_peak(pk, clk):
    """The bf16 peak matching the run's clock regime: MEASURED_PEAKS' burst figure when the
    median SM clock under load stayed within 5 % of the maximum (short runs at boost), its
    sustained figure (measured at a power-capped ~1.36 GHz median) otherwise."""
    mhz, mx = clk.get("sm_mhz"), clk.get("sm_max_mhz")
    burst = bool(mhz and mx and mhz >= 0.95 * mx)
    return (pk["bf16"] if burst else pk["bf16_sus"]), ("burst" if burst else "sustained")


# ------------------------------------------------------------------------ clocks -----------
class ClockSampler:
    NAMES = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x2: "applications_clocks_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self._nv = None
            self.err = str(e)
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM)
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                util = self._nv.nvmlDeviceGetUtilizationRates(self._h).gpu
                self.samples.append((mhz, r, util))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.02)

    def start(self):
        if self._nv:
            self._t.start()
        return self

    def stop(self):
        self._stop.set()
        if self._nv:
            self._t.join(timeout=1)
        busy = [s for s in self.samples if s[2] > 0] or self.samples
        reasons = set()
        for _, r, _ in busy:
            for bit, name in self.NAMES.items():
                if r & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median([s[0] for s in busy]) if busy else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons), "samples": len(busy)}


# ------------------------------------------------------------------------ oracle -----------
def oracle_step(a, T, seed):
    """One fwd+bwd of the oracle on T tokens of the workload (one rank, all E experts local)."""
    import synthetic as S
    from oracle import moe
    sh = S.LayerShape(T=T, d=a.d, f=a.f, E=a.experts, G=1, k=a.k, cf=a.cf, n_chunks=1)
    ins = S.gen_rank_inputs(seed, 0, sh, beta=a.beta)
    t0 = time.perf_counter()
    fwd = moe.forward([ins["x"]], ins["wg"], [ins["w1"]], [ins["w2"]], a.k, a.cf, a.chunks,
                      gate=a.gate)
    moe.backward(fwd, [ins["x"]], ins["wg"], [ins["w1"]], [ins["w2"]], [ins["dy"]])
    return time.perf_counter() - t0


def oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        n = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
        return int(n)
    except Exception:  # noqa: BLE001
        return os.cpu_count()


def calibrate_sample(a, budget_s):
    """Largest power-of-two token sample (>= 32) whose oracle fwd+bwd fits in ~budget_s s."""
    T = 64
    dt = oracle_step(a, T, a.seed)
    per_tok = dt / T
    Ts = 32
    while Ts * 2 <= a.tokens and per_tok * Ts * 2 <= budget_s:
        Ts *= 2
    return Ts, per_tok


def cpu_baseline(a, budget_s=15.0):
    Ts, _ = calibrate_sample(a, budget_s)
    dt = oracle_step(a, Ts, a.seed + 1)
    return {"value": Ts / dt, "unit": "tokens/s", "cores": oracle_threads(), "kind": "oracle",
            "sample": f"oracle fwd+bwd of {Ts} of the {a.tokens} tokens/GPU of the workload "
                      f"(one rank, all {a.experts} experts local), {dt:.1f} s, fp64 numpy "
                      f"matmuls + fp32 C gate, host cpu_count={os.cpu_count()}"}


def run_reference(a, world, rank):
    if rank != 0:
        return
    Ts, per_tok = calibrate_sample(a, 150.0 / max(1, a.steps + a.warmup))
    for i in range(a.warmup):
        oracle_step(a, Ts, a.seed + 10 + i)
    times = [oracle_step(a, Ts, a.seed + 100 + i) for i in range(a.steps)]
    ms = 1000.0 * statistics.mean(times)
    val = Ts / (ms / 1000.0)
    sample = (f"each step: oracle fwd+bwd of {Ts} tokens of the workload (one rank, all "
              f"{a.experts} experts local); fp64 numpy matmuls + fp32 C gate")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload(a, world),
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": oracle_threads(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------------------ GPU --------------
GEMM_OPS = ("expert_fc1", "expert_fc2", "expert_dfc2", "expert_dfc1", "expert_dw2", "expert_dw1")


def op_stats(tl, steps):
    tot = {}
    for r in tl:
        tot.setdefault(r["name"], [0.0, 0, set()])
        tot[r["name"]][0] += r["end_us"] - r["start_us"]
        tot[r["name"]][1] += 1
        tot[r["name"]][2].add(r["lane"])
    return {k: {"us_per_step": v[0] / steps, "launch_groups_per_step": v[1] / steps,
                "lanes": sorted(v[2])} for k, v in tot.items()}


def exposure_per_step(tl, steps):
    from paper_2404_19429_b200.lancet import exposed_comm_us
    d = exposed_comm_us(tl)
    return (d["exposed_us"] / steps / 1000.0, d["comm_us"] / steps / 1000.0,
            d["exposed_counts_us"] / steps / 1000.0, d["exposed_data_us"] / steps / 1000.0)


def run_e2e(a, world, ins, ctx, wg, w1, w2, dwg, dw1, dw2, dev, barrier, max_over_ranks):
    """End-to-end steps through the public API with HOST buffers.

    Every step copies its inputs x, dy from pinned host memory to the device and reads its
    results y, dx back to pinned host memory, inside the timed region.  Device inputs and
    outputs are triple-buffered and the copies run on their own streams, so the host->device
    copies of the next two steps and the device->host copies of earlier steps overlap the
    compute (a data-loader style pipeline: PCIe moves 64 MB each way per step, about as long
    as the step's compute, so a second step of slack absorbs the jitter); y's read-back
    overlaps the step's own backward."""
    import torch
    NB = 3
    bf = torch.bfloat16
    xh = torch.from_numpy(ins["x"]).to(bf).pin_memory()
    dyh = torch.from_numpy(ins["dy"]).to(bf).pin_memory()
    yh = [torch.empty(xh.shape, dtype=bf).pin_memory() for _ in range(NB)]
    dxh = [torch.empty(xh.shape, dtype=bf).pin_memory() for _ in range(NB)]
    xd = [torch.empty(xh.shape, dtype=bf, device=dev) for _ in range(NB)]
    dyd = [torch.empty(xh.shape, dtype=bf, device=dev) for _ in range(NB)]
    yd = [torch.empty(xh.shape, dtype=bf, device=dev) for _ in range(NB)]
    dxd = [torch.empty(xh.shape, dtype=bf, device=dev) for _ in range(NB)]
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev_in = [torch.cuda.Event() for _ in range(NB)]       # x landed (the forward waits on it)
    ev_in_dy = [torch.cuda.Event() for _ in range(NB)]    # dy landed (only the backward waits)
    ev_fwd = [torch.cuda.Event() for _ in range(NB)]
    ev_bwd = [torch.cuda.Event() for _ in range(NB)]
    ev_out = [torch.cuda.Event() for _ in range(NB)]

    def h2d(b):
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_bwd[b])            # buffer b's previous step is done with it
            xd[b].copy_(xh, non_blocking=True)
            ev_in[b].record(s_in)
            dyd[b].copy_(dyh, non_blocking=True)
            ev_in_dy[b].record(s_in)

    def run(n):
        for b in range(NB):
            ev_bwd[b].record(comp)
            ev_out[b].record(s_out)
        for j in range(min(NB - 1, n)):
            h2d(j)
        for i in range(n):
            b = i % NB
            comp.wait_event(ev_in[b])
            comp.wait_event(ev_out[b])            # host buffers of step i-NB have been read
            ctx.forward(xd[b], wg, w1, w2, a.k, a.cf, a.chunks, y=yd[b], routing=False)
            ev_fwd[b].record(comp)
            comp.wait_event(ev_in_dy[b])
            ctx.backward(dyd[b], dx=dxd[b], dwg=dwg, dw1=dw1, dw2=dw2)
            ev_bwd[b].record(comp)
            if i + NB - 1 < n:
                h2d((i + NB - 1) % NB)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_fwd[b])
                yh[b].copy_(yd[b], non_blocking=True)
                s_out.wait_event(ev_bwd[b])
                dxh[b].copy_(dxd[b], non_blocking=True)
                ev_out[b].record(s_out)

    run(2)
    torch.cuda.synchronize()
    barrier()
    ne = max(3, a.steps)

    def one_pass():
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(comp)
        s_in.wait_event(f0)
        h0 = time.perf_counter()
        run(ne)
        hms = (time.perf_counter() - h0) * 1000.0 / ne     # host enqueue time per step
        comp.wait_stream(s_out)
        f1.record(comp)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(f0.elapsed_time(f1) / ne), hms

    # three timed passes of K steps each (PCIe-bound, with more run-to-run spread than the
    # device-only number): the median is reported, all three are listed
    passes = [one_pass() for _ in range(3)]
    ems, host_ms = sorted(passes)[1]
    ok = bool(torch.equal(yh[(ne - 1) % NB], yd[(ne - 1) % NB].cpu()))
    nb = xh.numel() * xh.element_size()
    # the copies alone (no compute): the PCIe ceiling of this end-to-end loop
    def copy_ms(fn, reps=5):
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        c0.record(comp)
        for _ in range(reps):
            fn()
        c1.record(comp)
        torch.cuda.synchronize()
        return c0.elapsed_time(c1) / reps

    def h2d_only():
        xd[0].copy_(xh, non_blocking=True)
        dyd[0].copy_(dyh, non_blocking=True)

    def d2h_only():
        yh[0].copy_(yd[0], non_blocking=True)
        dxh[0].copy_(dxd[0], non_blocking=True)

    def both():
        with torch.cuda.stream(s_in):
            s_in.wait_stream(comp)
            h2d_only()
        with torch.cuda.stream(s_out):
            s_out.wait_stream(comp)
            d2h_only()
        comp.wait_stream(s_in)
        comp.wait_stream(s_out)

    h_ms, d_ms, b_ms = copy_ms(h2d_only), copy_ms(d2h_only), copy_ms(both)
    return {"value": world * a.tokens / (ems / 1000.0), "unit": "tokens/s",
            "h2d_bytes_per_step": 2 * nb, "d2h_bytes_per_step": 2 * nb, "ms_per_step": ems,
            "host_enqueue_ms_per_step": host_ms,
            "passes_ms_per_step": [round(p_[0], 4) for p_ in passes], "reported": "median of the passes",
            "host_affinity": getattr(a, "cpu_affinity", None),
            "readback_checked": ok,
            "copies_alone_ms": {"h2d": h_ms, "d2h": d_ms, "both_directions": b_ms,
                                "h2d_gbs": 2 * nb / (h_ms * 1e6), "d2h_gbs": 2 * nb / (d_ms * 1e6)},
            "path": "pinned host x, dy -> device (own stream) -> lancet_moe_forward + lancet_moe_backward "
                    "(C-ABI) -> y, dx -> pinned host (own stream); device buffers triple-buffered so "
                    "copies overlap neighbouring steps' compute; every step's copies are inside the "
                    "timed region (first H2D to last D2H)"}


def measure_arm(a, ctx, lancet, flags, step, stream, barrier, max_over_ranks, n_chunks):
    """One exchange arm measured on one definition, all ranks' max:
      ms_per_step          clean pass (no per-op events), the throughput number;
      exposed_a2a_ms       instants where an exchange op (lane 1) runs and no compute op does,
                           from per-op events of a second pass;
      unoverlapped_a2a_ms  the lane-1 time of the serial schedule (one stream, chunks merged,
                           dW after the exchanges: LANCET_FLAG_SERIAL);
      no_comm_ms_per_step  the same schedule with the data exchanges skipped (LANCET_FLAG_NO_COMM,
                           timing only), so ms_per_step - no_comm bounds the exposed exchange
                           time from above (it also removes the exchanges' SM / HBM contention).
    In the push mode the lane-1 ops are the fused token kernels (permute / gather work
    included); NO_COMM keeps that local work (same kernels on local buffers) so the
    differential is comparable across push, pull and NCCL."""
    import torch

    def run(fl, n, instrumented=False):
        ctx.set_flags(fl | (lancet.FLAG_TIMELINE if instrumented else 0))
        for _ in range(2):
            step(n_chunks)
        torch.cuda.synchronize()
        if instrumented:
            ctx.timeline_begin(stream)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            step(n_chunks)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = max_over_ranks(e0.elapsed_time(e1) / n)
        return ms, (ctx.timeline(cap=200000) if instrumented else None)

    ctx.set_flags(flags)
    for _ in range(a.warmup):
        step(n_chunks)
    steps = max(3, a.steps)
    ms, _ = run(flags, steps)
    ms_instr, tl = run(flags, steps, True)
    exposed, comm, exp_c, exp_d = exposure_per_step(tl, steps)
    ns = max(3, min(10, steps))
    ms_serial, tls = run(flags | lancet.FLAG_SERIAL, ns, True)
    unover = sum(r["end_us"] - r["start_us"] for r in tls if r["lane"] == 1) / ns / 1000.0
    ms_nocomm, _ = run(flags | lancet.FLAG_NO_COMM, steps)
    ms_serial_clean, _ = run(flags | lancet.FLAG_SERIAL, steps)
    ctx.set_flags(flags)
    world = ctx.world
    from paper_2404_19429_b200.chunk_tuner import profile_ops
    return {"n_chunks": n_chunks, "ms_per_step": ms, "tokens_per_s": world * a.tokens / (ms / 1000.0),
            "op_profile_us": [round(v, 3) for v in profile_ops(tl, steps, n_chunks)],
            "instrumented_ms_per_step": ms_instr,
            "exposed_a2a_ms": max_over_ranks(exposed), "a2a_ms_on_comm_lane": max_over_ranks(comm),
            "exposed_a2a_split_ms": {"counts": exp_c, "data": exp_d},
            "unoverlapped_a2a_ms": max_over_ranks(unover),
            "exposed_over_unoverlapped": (max_over_ranks(exposed) / max_over_ranks(unover)) if unover > 0 else None,
            "serial_ms_per_step": ms_serial_clean,
            "no_comm_ms_per_step": ms_nocomm, "exposed_upper_bound_ms": ms - ms_nocomm}


def tuner_record(a, ctx, lancet, flags, step_fn, stream, barrier, max_over_ranks, schedule, bytes_full,
                 ns=(1, 2, 4, 8), fit_on=(1, 4)):
    """Every n of `ns` measured on one definition (measure_arm), and the chunk-count tuner
    (lancet_tune_chunks, NEXT-3) fitted on the op profiles of `fit_on` predicting n = 1..8:
    predicted vs measured step time per n, the tuner's pick and the measured best."""
    from paper_2404_19429_b200.chunk_tuner import tune
    import numpy as np
    by_n = [measure_arm(a, ctx, lancet, flags, step_fn, stream, barrier, max_over_ranks, n) for n in ns]
    prof = {r["n_chunks"]: np.array(r["op_profile_us"]) for r in by_n if r["n_chunks"] in fit_on}
    best, pred, expo = tune(prof, bytes_full, schedule, max_chunks=max(8, max(ns)))
    meas = {r["n_chunks"]: r["ms_per_step"] * 1000.0 for r in by_n}
    pts = [{"n": n, "measured_us": meas[n], "predicted_us": float(pred[n - 1]),
            "error": float((pred[n - 1] - meas[n]) / meas[n]), "predicted_exposed_us": float(expo[n - 1])}
           for n in ns]
    return {"by_n": by_n,
            "tuner": {"schedule": "push pipeline" if schedule == 1 else "per-chunk launches",
                      "profiled_n": sorted(prof), "predicted_us_n1_to_8": [round(float(v), 1) for v in pred],
                      "points": pts, "mean_abs_error": float(np.mean([abs(p["error"]) for p in pts])),
                      "pick": int(best), "measured_best": int(min(meas, key=meas.get)),
                      "model": "DP over partition counts (P:L405-L414) scored by the two-lane stage "
                               "simulator (P:L488-L499) on lancet.cu's schedule; ops from the per-op "
                               "timelines at the profiled n (caching profiler, P:L322-L323); exchanges "
                               "from the size-interpolated cost model at C/n (P:L325-L328)"}}


BLOCK_OPS_NONMOE = ("ln1", "qkv_proj", "attention", "o_proj", "ln2")


def block_record(a, world, rank, local_rank, stream, barrier, max_over_ranks, ns=(1, 2, 4, 8), experts=32):
    """BASELINE configs[3]: the full GPT-MoE block (pre-LN GPT-2 block with the MoE layer as its
    MLP) forward with Lancet's pre-MoE partition (fig:part_all), per
    GPU: 8 sequences x 1024 tokens, d_model 2048, 16 heads, ffn 8192, 32 experts (32/N per GPU),
    Switch top-1, cf 1.25.  Per chunk count n: the pipelined forward (clean pass), its exposed /
    unoverlapped exchange time (instrumented pass; LANCET_FLAG_SERIAL = one stream, chunks
    merged, no overlap) and the no-comm differential; per-op times of the n = 4 pass and the
    attention kernel's roofline."""
    import dataclasses
    import torch
    import synthetic as S
    from paper_2404_19429_b200 import block as B
    from paper_2404_19429_b200 import lancet
    sh = S.BlockShape(n_seq=8, seq_len=1024, d=2048, n_heads=16, f=8192, E=experts, G=world, k=1, cf=1.25, n_chunks=4)
    ins = S.gen_block_rank_inputs(a.seed + 7, rank, sh, beta=a.beta, with_dy=False)
    dev = torch.device("cuda", local_rank)
    bf = torch.bfloat16
    p = {key: torch.from_numpy(ins[key]).to(dev, torch.float32 if key in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "wg")
                                            else bf) for key in B.PARAMS}
    x = torch.from_numpy(ins["x"]).to(dev, bf)
    del ins
    out = torch.empty_like(x)
    moe = lancet.LayerConfig(d_model=sh.d, d_ffn=sh.f, n_experts=sh.E, max_tokens=sh.T, max_k=sh.k, max_chunks=8)
    import torch.distributed as dist
    blk = B.Block(B.BlockConfig(moe, n_heads=sh.n_heads, seq_len=sh.seq_len, max_capacity_factor=sh.cf),
                  world=world, rank=rank, device=local_rank, pg=dist.group.WORLD if world > 1 else None)
    base = blk.moe.cfg.flags

    dout = torch.randn(x.shape, generator=torch.Generator(device=dev).manual_seed(a.seed + 8), device=dev).to(bf)

    def one(n, bwd):
        blk.forward(x, p, sh.k, sh.cf, n, out=out)
        if bwd:
            blk.backward(dout)

    def run(n, fl, steps, instrumented=False, bwd=False):
        blk.moe.set_flags(base | fl | (lancet.FLAG_TIMELINE if instrumented else 0))
        for _ in range(3):
            one(n, bwd)
        torch.cuda.synchronize()
        if instrumented:
            blk.moe.timeline_begin(stream)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            one(n, bwd)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / steps), (blk.moe.timeline(cap=200000) if instrumented else None)

    steps = max(5, min(a.steps, 30))
    for _ in range(max(3, min(a.warmup, 20))):
        blk.forward(x, p, sh.k, sh.cf, 4, out=out)
    by_n, ops4, opsb = [], None, None
    for n in ns:
        ms, _ = run(n, 0, steps)
        _, tl = run(n, 0, steps, True)
        exposed, comm, _, _ = exposure_per_step(tl, steps)
        _, tls = run(n, lancet.FLAG_SERIAL, 3, True)
        unover = sum(r["end_us"] - r["start_us"] for r in tls if r["lane"] == 1) / 3 / 1000.0
        ms_serial, _ = run(n, lancet.FLAG_SERIAL, steps)
        ms_nocomm, _ = run(n, lancet.FLAG_NO_COMM, steps)
        ms_fb, _ = run(n, 0, steps, bwd=True)
        by_n.append({"n_chunks": n, "ms_per_step": ms, "tokens_per_s": world * sh.T / (ms / 1000.0),
                     "fwd_bwd_ms_per_step": ms_fb, "fwd_bwd_tokens_per_s": world * sh.T / (ms_fb / 1000.0),
                     "exposed_a2a_ms": max_over_ranks(exposed), "a2a_ms_on_comm_lane": max_over_ranks(comm),
                     "unoverlapped_a2a_ms": max_over_ranks(unover), "serial_ms_per_step": ms_serial,
                     "no_comm_ms_per_step": ms_nocomm, "exposed_upper_bound_ms": ms - ms_nocomm})
        if n == 4:
            ops4 = op_stats(tl, steps)
            _, tlb = run(n, 0, steps, True, bwd=True)
            opsb = op_stats(tlb, steps)
    blk.moe.set_flags(base)
    # a stack of two blocks (same parameters, own buffers): consecutive forwards vs the chunk
    # pipeline across the blocks (lancet_block_forward_stack: block 2's chunk c starts once block
    # 1 has combined chunk c)
    blk2 = B.Block(B.BlockConfig(moe, n_heads=sh.n_heads, seq_len=sh.seq_len, max_capacity_factor=sh.cf),
                   world=world, rank=rank, device=local_rank, pg=dist.group.WORLD if world > 1 else None)
    out2 = [torch.empty_like(x), torch.empty_like(x)]
    stack = []
    for n in (1, 2, 4):
        def cons():
            blk.forward(x, p, sh.k, sh.cf, n, out=out2[0])
            blk2.forward(out2[0], p, sh.k, sh.cf, n, out=out2[1])

        def pipe():
            B.forward_stack([blk, blk2], x, [p, p], sh.k, sh.cf, n, outs=out2)
        tm = {}
        for name, fn in (("consecutive", cons), ("stack_pipelined", pipe)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            tm[name] = max_over_ranks(e0.elapsed_time(e1) / steps)
        stack.append({"n_chunks": n, "consecutive_ms": tm["consecutive"], "stack_ms": tm["stack_pipelined"]})
    blk2.close()
    best = min(by_n, key=lambda r: r["ms_per_step"])
    pk = peaks()
    # attention: algorithmic causal FLOPs 2 * 2 * S^2 / 2 * hd per (sequence, head); the kernel
    # also recomputes Q K^T (two-pass exact softmax) and evaluates 2 exp2 per unmasked score
    att_flops = sh.n_seq * sh.n_heads * 2.0 * sh.seq_len ** 2 * (sh.d // sh.n_heads)
    att_us = ops4["attention"]["us_per_step"] if ops4 and "attention" in ops4 else None
    proj_flops = 2.0 * sh.T * sh.d * (3 * sh.d) + 2.0 * sh.T * sh.d * sh.d
    proj_us = sum(ops4[o]["us_per_step"] for o in ("qkv_proj", "o_proj") if ops4 and o in ops4) or None
    rec = {
        "workload": f"GPT-MoE block forward (BASELINE configs[3]): {sh.n_seq}x{sh.seq_len} tokens/GPU, d_model={sh.d}, "
                    f"{sh.n_heads} heads, ffn={sh.f}, experts={sh.E} ({sh.E // world}/GPU), Switch top-1, cf={sh.cf}, "
                    f"bf16; MoE over the peer push transport" + (" (one-rank group: exchanges to self)" if world == 1 else ""),
        "metric": "block forward tokens/s (fwd_bwd_value: forward + backward); exposed all-to-all ms/iter",
        "unit": "tokens/s",
        "value": world * sh.T / (best["ms_per_step"] / 1000.0), "best_n_chunks": best["n_chunks"],
        "by_n": by_n,
        "ops_us_per_step_n4": {o: round(v["us_per_step"], 2) for o, v in (ops4 or {}).items()},
        "fwd_bwd_ops_us_per_step_n4": {o: round(v["us_per_step"], 2) for o, v in (opsb or {}).items()},
        "fwd_bwd_value": world * sh.T / (min(r["fwd_bwd_ms_per_step"] for r in by_n) / 1000.0),
        "two_block_stack_forward": stack,
        "attention_roofline": {
            "bound": "tensor", "achieved": att_flops / (att_us * 1e-6) / 1e12 if att_us else None,
            "peak": pk["bf16_sus"], "unit": "TFLOP/s",
            "frac": (att_flops / (att_us * 1e-6) / 1e12 / pk["bf16_sus"]) if att_us else None,
            "flops": att_flops, "us": att_us,
            "note": "algorithmic causal FLOPs (QK^T and PV on the unmasked half) / summed event time of the "
                    "per-chunk attention launches (n = 4, instrumented pass); the two-pass kernel executes 1.5x "
                    "the MMA work and 2 exp2 per score on the SFU"},
        "projection_gemms": {"achieved_tflops": proj_flops / (proj_us * 1e-6) / 1e12 if proj_us else None,
                             "us": proj_us, "flops": proj_flops},
    }
    blk.close()
    return rec


def make_context(a, lancet, cfg, world, rank, local_rank, dev):
    """transport auto (world > 1): the copy-engine peer transport when every rank can set it up
    (CUDA IPC between all ranks' devices, stream memory operations), else NCCL -- decided
    collectively so all ranks use the same one."""
    import torch
    import torch.distributed as dist
    import dataclasses
    pg = dist.group.WORLD if world > 1 else None
    # the push mode of the peer transport is fixed at creation (every exchange fused into the
    # token kernels, no host synchronisation)
    pcfg = dataclasses.replace(cfg, flags=cfg.flags | (0 if a.no_push else lancet.FLAG_PEER_PUSH))
    if a.transport != "auto":
        a.transport_used = a.transport
        return lancet.Context(pcfg if a.transport == "peer" else cfg, world=world, rank=rank, device=local_rank,
                              pg=pg, transport=a.transport)
    if world == 1:
        a.transport_used = "none"
        return lancet.Context(cfg, world=1, rank=0, device=local_rank)
    ctx, ok = None, 1.0
    try:
        ctx = lancet.Context(pcfg, world=world, rank=rank, device=local_rank, pg=pg, transport="peer")
    except Exception as e:  # noqa: BLE001
        print(f"rank {rank}: peer transport unavailable ({e}); voting for NCCL", file=sys.stderr)
        ok = 0.0
    t = torch.tensor([ok], dtype=torch.float64, device="cpu" if a.same_device else dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if t.item() == 1.0:
        a.transport_used = "peer"
        return ctx
    if ctx is not None:
        ctx.close()
    a.transport_used = "nccl"
    return lancet.Context(cfg, world=world, rank=rank, device=local_rank, pg=pg, transport="nccl")


def gpu_local_cpus(local_rank):
    """The CPUs NVML reports as closest to this GPU (its NUMA node), or None."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local_rank)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:  # noqa: BLE001
        return None


def run_lancet(a, world, rank, local_rank):
    import torch
    import torch.distributed as dist
    import synthetic as S
    from paper_2404_19429_b200 import build, lancet
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    # host threads (and with them the pinned buffers of the end-to-end loop, first-touch) on
    # the GPU's own NUMA node: on a multi-socket host, DMA to a far socket's memory crosses the
    # socket link (the pool's boxes are single-node VMs, where this is a no-op; their two-way
    # copy time still varies between runs, 1.36-1.83 ms per step, hence the median of passes)
    a.cpu_affinity = None
    a.cpu_affinity_all = os.sched_getaffinity(0)
    if not os.environ.get("LANCET_BENCH_NO_AFFINITY"):
        cpus = gpu_local_cpus(local_rank)
        if cpus:
            os.sched_setaffinity(0, cpus)
            a.cpu_affinity = f"{len(cpus)} CPUs local to GPU {local_rank} (NVML)"
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    E_l = a.experts // world
    sh = S.LayerShape(T=a.tokens, d=a.d, f=a.f, E=a.experts, G=world, k=a.k, cf=a.cf, n_chunks=a.chunks)
    ins = S.gen_rank_inputs(a.seed, rank, sh, beta=a.beta)
    bf = torch.bfloat16
    x = torch.from_numpy(ins["x"]).to(dev, bf)
    wg = torch.from_numpy(ins["wg"]).to(dev)
    w1 = torch.from_numpy(ins["w1"]).to(dev, bf)
    w2 = torch.from_numpy(ins["w2"]).to(dev, bf)
    dy = torch.from_numpy(ins["dy"]).to(dev, bf)
    # the timed region runs without per-op events (they cost ~5 % of the step: every event
    # record between two kernels is a stream operation that also breaks programmatic dependent
    # launch); the per-op breakdown, the GEMM roofline and the exposure come from a second,
    # instrumented pass of the same K steps right after it
    flags = a.flags & ~lancet.FLAG_TIMELINE
    if a.gate == "bpr":
        flags |= lancet.FLAG_GATE_BPR
    elif a.gate == "random":
        flags |= lancet.FLAG_GATE_RANDOM
    cfg = lancet.LayerConfig(d_model=a.d, d_ffn=a.f, n_experts=a.experts, max_tokens=a.tokens,
                             max_k=a.k, max_chunks=max(8, a.chunks), dtype="bf16", flags=flags)
    ctx = make_context(a, lancet, cfg, world, rank, local_rank, dev)
    if a.transport_used == "peer" and not a.no_push:
        flags |= lancet.FLAG_PEER_PUSH
    stream = torch.cuda.current_stream()
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    dwg = torch.empty_like(wg)
    dw1 = torch.empty(w1.shape, dtype=torch.float32, device=dev)
    dw2 = torch.empty(w2.shape, dtype=torch.float32, device=dev)

    def step(xx=x, dyy=dy):
        ctx.forward(xx, wg, w1, w2, a.k, a.cf, a.chunks, y=y, routing=False)
        ctx.backward(dyy, dx=dx, dwg=dwg, dw1=dw1, dw2=dw2)

    def step_on(c):
        def f(n):
            c.forward(x, wg, w1, w2, a.k, a.cf, n, y=y, routing=False)
            c.backward(dy, dx=dx, dwg=dwg, dw1=dw1, dw2=dw2)
        return f

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if a.same_device else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if a.only_block:
        clocks = ClockSampler(local_rank).start()
        rec = block_record(a, world, rank, local_rank, torch.cuda.current_stream(), barrier, max_over_ranks)
        if world == 1:
            rec["ep8_expert_shapes"] = block_record(a, world, rank, local_rank, torch.cuda.current_stream(), barrier,
                                                    max_over_ranks, experts=4)
        rec["clocks"] = clocks.stop()
        if rank == 0:
            print(json.dumps({"block": rec}), flush=True)
        ctx.close()
        return

    # chunk count: auto at N > 1 = the fastest of n = 1, 2, 4, 8 over a short probe (max over
    # ranks); the single-GPU path has no exchange and runs unchunked whatever n says
    ep_path = world > 1 or bool(flags & lancet.FLAG_FORCE_EP) or a.transport == "peer"
    n_probe = None
    if a.chunks_req <= 0:
        if ep_path:
            n_probe = {}
            for n in (1, 2, 4, 8):
                a.chunks = n
                for _ in range(2):
                    step()
                barrier()
                torch.cuda.synchronize()
                p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                p0.record(stream)
                for _ in range(5):
                    step()
                p1.record(stream)
                torch.cuda.synchronize()
                n_probe[n] = max_over_ranks(p0.elapsed_time(p1) / 5)
            a.chunks = min(n_probe, key=n_probe.get)
        else:
            a.chunks = 1
    clocks = ClockSampler(local_rank).start()
    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()

    def timed(instrumented):
        ctx.set_flags(flags | (lancet.FLAG_TIMELINE if instrumented else 0))
        if instrumented:
            step()                                        # one step to settle the event pool
            torch.cuda.synchronize()
            ctx.timeline_begin(stream)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        for _ in range(a.steps):
            step()
        host = (time.perf_counter() - h0) * 1000.0 / a.steps    # host enqueue time per step
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / a.steps), host

    # ---- timed region (device time, CUDA events on the caller stream) -------------------
    ms, host_ms = timed(False)
    clk = clocks.stop()
    gemm_ops = {}
    if not a.no_timeline:
        # roofline pass: events around the six GEMM launches only (least perturbation)
        flags_saved = flags
        flags = flags | lancet.FLAG_TIMELINE_GEMM_ONLY
        timed(True)
        gemm_ops = op_stats(ctx.timeline(cap=200000), a.steps)
        flags = flags_saved
    ms_instr, _ = timed(not a.no_timeline)          # full per-op breakdown and exposure
    tl = ctx.timeline(cap=200000) if not a.no_timeline else []
    ctx.set_flags(flags)
    ops = op_stats(tl, a.steps)
    f_l, b_l = ctx.launch_counts()
    send, recv, C = ctx.counts(a.chunks)
    rows_expert = int(recv.sum())                     # rows this rank's experts processed
    ep = world > 1 or bool(flags & lancet.FLAG_FORCE_EP) or a.transport == "peer"   # a2a on
    exposed_ms, comm_ms, exp_counts_ms, exp_data_ms = exposure_per_step(tl, a.steps) if ep else (0.0,) * 4
    exposed_ms = max_over_ranks(exposed_ms)

    # ---- unoverlapped baseline (world > 1): serial schedule, one stream, chunks merged -------
    unoverlapped_ms = 0.0
    if ep:
        ctx.set_flags(flags | lancet.FLAG_SERIAL | lancet.FLAG_TIMELINE)
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        ctx.timeline_begin(stream)
        barrier()
        ns = max(3, min(10, a.steps))
        for _ in range(ns):
            step()
        torch.cuda.synchronize()
        tls = ctx.timeline(cap=200000)
        unoverlapped_ms = max_over_ranks(
            sum(r["end_us"] - r["start_us"] for r in tls if r["lane"] == 1) / ns / 1000.0)
        ctx.set_flags(flags)

    # ---- end to end through the public API with host buffers ---------------------------------
    e2e = None
    if not a.no_e2e:
        e2e = run_e2e(a, world, ins, ctx, wg, w1, w2, dwg, dw1, dw2, dev, barrier, max_over_ranks)

    # ---- roofline of the dominant kernel (the tcgen05 grouped GEMM, 6 launches per step) ----
    pk = peaks()
    peak, regime = gemm_peak(pk, clk)
    gsrc = gemm_ops or ops
    gemm_us = sum(gsrc[o]["us_per_step"] for o in GEMM_OPS if o in gsrc)
    gemm_flops = 12.0 * rows_expert * a.d * a.f       # algorithmic: admitted rows only
    achieved = gemm_flops / (gemm_us * 1e-6) / 1e12 if gemm_us > 0 else 0.0
    # DRAM bytes of the six GEMM launches from the committed `ncu --set full` capture -- only
    # when this run is the captured configuration (world 1, configs[1] shape, Switch gate)
    traffic, traffic_src = None, "no ncu capture of this configuration"
    prof = os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            want = {"tokens": a.tokens, "d": a.d, "f": a.f, "experts": a.experts, "k": a.k, "world": world,
                    "gate": a.gate, "cf": a.cf}
            if all(pj.get("config", {}).get(key) == v for key, v in want.items()):
                traffic = pj.get("dram_bytes_per_step")
                traffic_src = f"{pj.get('source')} (dram__bytes_read.sum + dram__bytes_write.sum, six launches)"
        except Exception:  # noqa: BLE001
            traffic = None
    kernels = {}
    for o in GEMM_OPS:
        if o in gsrc and gsrc[o]["us_per_step"] > 0:
            kernels[o] = {"us": gsrc[o]["us_per_step"],
                          "tflops": 2.0 * rows_expert * a.d * a.f / (gsrc[o]["us_per_step"] * 1e-6) / 1e12}
    # memory-bound kernels: algorithmic bytes per step
    tk = a.tokens * a.k
    adm = int(send.sum())
    rowb = a.d * 2
    mem_bytes = {
        "gate": a.tokens * rowb + a.tokens * (a.experts * 4 + a.k * 8),
        "permute": a.tokens * rowb + adm * rowb,
        "combine": adm * rowb + a.tokens * rowb,
        "combine_bwd": a.tokens * rowb + 2 * adm * rowb,
        "unpermute_gate_bwd": adm * rowb + a.tokens * rowb,
        "gate_dwg": a.tokens * rowb + a.tokens * a.experts * 4,
    }
    for o, b in mem_bytes.items():
        if o in ops and ops[o]["us_per_step"] > 0:
            if 2 in ops[o]["lanes"]:
                # side stream: the event span runs concurrently with the GEMMs (sharing SMs and
                # waiting for them); it is not the kernel's duration, so no bandwidth is derived
                # from it (isolated durations: the ncu launch list under profiles/)
                kernels[o] = {"span_us": ops[o]["us_per_step"],
                              "note": "side stream, concurrent with the expert GEMMs: event span, "
                                      "not an isolated duration"}
                continue
            kernels[o] = {"us": ops[o]["us_per_step"],
                          "gbs": b / (ops[o]["us_per_step"] * 1e-6) / 1e9,
                          "hbm_frac": b / (ops[o]["us_per_step"] * 1e-6) / 1e9 / pk["hbm"]}
            if o == "gate":
                kernels[o]["note"] = ("event span of K1 + K2 (gate, slot scan and the histogram "
                                      "memset); bytes are the gate's")
    # isolated durations of the same kernels from the committed ncu capture (cold cache,
    # serialised, --clock-control none): the in-step event spans above include launch gaps
    # and lose programmatic dependent launch at every event record
    iso = os.path.join(ROOT, "profiles", "ncu_simt_traffic.json")
    if os.path.exists(iso) and a.tokens == 16384 and a.experts == 8 and a.d == 1024:
        try:
            launches = json.load(open(iso))["launches"]
            names = {"gate": ["gate_stream"], "permute": ["permute_kernel"], "combine": ["combine_kernel"],
                     "combine_bwd": ["combine_bwd"], "unpermute_gate_bwd": ["k6_stream"],
                     "gate_dwg": ["dwg_stream", "dwg_reduce4"]}
            for o, pats in names.items():
                if o not in kernels or o not in mem_bytes:
                    continue
                us = []
                for pat in pats:
                    m = [l["us"] for l in launches if pat in l["kernel"] and
                         not (pat == "combine_kernel" and "bwd" in l["kernel"])]
                    if m:
                        us.append(min(m))
                if len(us) == len(pats):
                    t = sum(us)
                    kernels[o]["ncu_isolated_us"] = t
                    kernels[o]["hbm_frac_isolated"] = mem_bytes[o] / (t * 1e-6) / 1e9 / pk["hbm"]
        except Exception:  # noqa: BLE001
            pass
    for o, v in ops.items():
        if o not in kernels:
            kernels[o] = {"us": v["us_per_step"]}
    del tk

    out = {
        "metric": METRIC, "value": world * a.tokens / (ms / 1000.0), "unit": "tokens/s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded; synthetic/ recipe, DESIGN.md)",
        "config": workload(a, world),
        "n_chunks_used": a.chunks if ep_path else 1,
        "n_chunks_note": ("the fastest of a 5-step probe per n (max over ranks, ms per step): "
                          + json.dumps({str(k_): round(v_, 4) for k_, v_ in n_probe.items()})
                          if n_probe else
                          ("set by --chunks" if ep_path else
                           "single GPU: no exchange to pipeline, the layer runs unchunked; the "
                           "'ep' record measures n = 1, 2, 4, 8 over a one-rank group")),
        "host_enqueue_ms_per_step": host_ms,
        "instrumented_ms_per_step": ms_instr,
        "exposed_a2a_ms": exposed_ms, "a2a_ms_on_comm_lane": comm_ms,
        "exposed_a2a_split_ms": {"counts": exp_counts_ms, "data": exp_data_ms},
        "unoverlapped_a2a_ms": unoverlapped_ms,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_regime": regime, "peak_burst": pk["bf16"], "peak_sustained": pk["bf16_sus"],
                     "frac_burst": achieved / pk["bf16"], "frac_sustained": achieved / pk["bf16_sus"],
                     "kernel": "tc_gemm_kernel (tcgen05 grouped GEMM), 6 launches/step; "
                               "achieved = 12*rows*d*f algorithmic FLOP / summed CUDA-event time "
                               "of the six launches, from events around the GEMM launches only "
                               "over a second pass of the same K steps (the clean timed pass "
                               "carries no per-op events)",
                     "peak_source": pk["src"] + (" bf16_tflops (median SM clock >= 0.95 x max)" if regime == "burst"
                                                 else " bf16_tflops_sustained (median SM clock < 0.95 x max)")},
        "kernels": kernels,
        "launch_groups": {o: v["launch_groups_per_step"] for o, v in ops.items()},
        "gpu_launches": (f_l + b_l) * a.steps,
        "clocks": clk,
        "routing": {"capacity": C, "admitted_pairs": adm, "dropped_pairs": a.tokens * a.k - adm,
                    "expert_rows_this_rank": rows_expert},
    }
    if e2e:
        out["e2e"] = e2e
    if world > 1:
        out["exposure_definition"] = ("lane 1 = exchange ops; " + (
            "push mode: the fused token kernels (permute / gather work included)" if a.transport_used == "peer"
            and not a.no_push else "copies / NCCL kernels only"))
    import dataclasses
    if world == 1 and not a.no_ep:
        # the expert-parallel chunk pipeline (S1 / S2) on this GPU: a one-rank group of the peer
        # transport in push mode -- every exchange of the N > 1 path is executed (to self), so
        # the line carries the metric's second half (exposed vs unoverlapped all-to-all)
        pcfg = dataclasses.replace(cfg, flags=(flags & ~lancet.FLAG_FORCE_EP) | lancet.FLAG_PEER_PUSH)
        try:
            ectx = lancet.Context(pcfg, world=1, rank=0, device=local_rank, transport="peer")
            ep_flags = pcfg.flags
            rec = tuner_record(a, ectx, lancet, ep_flags, step_on(ectx), stream, barrier, max_over_ranks, 1,
                               float(adm * rowb), ns=sorted({1, 2, 4, 8, a.chunks}))
            out["ep"] = {"transport": "peer push, one-rank group (all exchanges to self)", **rec}
            ectx.close()
        except Exception as ex:  # noqa: BLE001 -- an auxiliary record never costs the headline line
            out["ep"] = {"error": f"{type(ex).__name__}: {ex}"}
    if world > 1 and not a.no_arms:
        # every transport on the same definitions (push / pull over the peer transport, NCCL)
        arms = {}
        for name in ("push", "pull", "nccl"):
            if name != "nccl" and a.transport_used != "peer":
                continue
            if name == "nccl" and a.same_device:
                arms[name] = {"skipped": "NCCL refuses several ranks on one device (--same-device)"}
                continue
            actx, own = ctx, False
            try:
                if not (name == ("push" if not a.no_push else "pull") and a.transport_used == "peer"):
                    acfg = dataclasses.replace(cfg, flags=flags & ~lancet.FLAG_PEER_PUSH | (lancet.FLAG_PEER_PUSH if name == "push" else 0))
                    actx = lancet.Context(acfg, world=world, rank=rank, device=local_rank,
                                          pg=dist.group.WORLD, transport="nccl" if name == "nccl" else "peer")
                    own = True
                afl = flags & ~lancet.FLAG_PEER_PUSH | (lancet.FLAG_PEER_PUSH if name == "push" else 0)
                arms[name] = measure_arm(a, actx, lancet, afl, step_on(actx), stream, barrier, max_over_ranks, a.chunks)
            except Exception as ex:  # noqa: BLE001 -- an auxiliary record never costs the headline line
                arms[name] = {"error": f"{type(ex).__name__}: {ex}"}
            if own:
                barrier()
                actx.close()
        out["arms"] = arms
        # the chunk-count tuner on the main arm: n = 1, 2, 4, 8 measured, predicted from n = 1, 4
        sched = 1 if (a.transport_used == "peer" and not a.no_push) else 0
        try:
            out["chunk_tuner"] = tuner_record(a, ctx, lancet, flags, step_on(ctx), stream, barrier, max_over_ranks,
                                              sched, float(adm * rowb))["tuner"]
        except Exception as ex:  # noqa: BLE001
            out["chunk_tuner"] = {"error": f"{type(ex).__name__}: {ex}"}
    if not a.no_block:
        try:
            out["block"] = block_record(a, world, rank, local_rank, stream, barrier, max_over_ranks)
        except Exception as ex:  # noqa: BLE001
            out["block"] = {"error": f"{type(ex).__name__}: {ex}"}
        if world == 1 and "error" not in out["block"]:
            # the per-GPU expert shapes of the 8-GPU run (4 local experts receiving 8192 rows per
            # step) on this GPU: the same block with E = 4 experts in a one-rank group -- with
            # E_l = 32 every chunk splits each expert's ~256 rows into tiny GEMM groups
            try:
                out["block"]["ep8_expert_shapes"] = block_record(a, world, rank, local_rank, stream, barrier,
                                                                 max_over_ranks, experts=4)
            except Exception as ex:  # noqa: BLE001
                out["block"]["ep8_expert_shapes"] = {"error": f"{type(ex).__name__}: {ex}"}
    if rank == 0 and not a.no_cpu_baseline:
        os.sched_setaffinity(0, a.cpu_affinity_all)    # the oracle gets every host core again
        out["cpu_baseline"] = cpu_baseline(a)
    barrier()
    if rank == 0:
        print(json.dumps(out), flush=True)
    barrier()
    ctx.close()


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus and rank == 0:
        print(f"warning: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    if a.experts % world:
        raise SystemExit("experts must be divisible by the number of GPUs")
    if a.impl == "reference":
        run_reference(a, world, rank)
        return
    import torch
    import torch.distributed as dist
    if a.same_device:
        local_rank = 0
    if world > 1:
        torch.cuda.set_device(local_rank)
        if a.same_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_lancet(a, world, rank, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
