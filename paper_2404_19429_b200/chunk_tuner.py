"""Chunk-count tuner: the binding of lancet_tune_chunks
(include/lancet_moe.h, csrc/tuner.cpp) plus the caching op profiler that feeds it.

Lancet picks the number of partitions with a DP over partition ranges scored by a pipeline
scheduler from profiled op costs and a communication cost model
interpolated over message sizes with the C/n approximation (L322-L328).  For one MoE layer the
DP is a scan over n; the simulation runs in the library (the schedule lancet.cu enqueues), and
this module only marshals: `profile_ops` turns the per-op timeline of one step at a profiled
chunk count into per-chunk op costs, `tune` calls the library.
"""
from __future__ import annotations

import ctypes

import numpy as np

from .lancet import _check, load_library

OPS = ("GATE", "COUNTS", "DISPATCH", "FC1", "FC2", "COMBINE", "GATHER", "K5", "BWD_DISPATCH", "DFC2", "DFC1",
       "DW", "BWD_COMBINE", "K6", "K7")
N_OPS = len(OPS)
ONCE = ("GATE", "COUNTS", "K7")

# timeline op names (lancet.cu OpScope) -> op kind of the tuner
TIMELINE_TO_OP = {
    "gate": "GATE", "permute": "GATE", "a2a_counts": "COUNTS",
    "a2a_dispatch": "DISPATCH", "a2a_dispatch_push": "DISPATCH",
    "expert_fc1": "FC1", "expert_fc2": "FC2",
    "a2a_combine": "COMBINE", "a2a_combine_fused": "COMBINE", "combine": "GATHER",
    "combine_bwd": "K5", "a2a_bwd_dispatch": "BWD_DISPATCH", "a2a_bwd_dispatch_push": "BWD_DISPATCH",
    "expert_dfc2": "DFC2", "expert_dfc1": "DFC1", "expert_dw2": "DW", "expert_dw1": "DW",
    "a2a_bwd_combine": "BWD_COMBINE", "a2a_bwd_combine_fused": "BWD_COMBINE",
    "unpermute_gate_bwd": "K6", "gate_dwg": "K7",
}


class _TuneInput(ctypes.Structure):
    _fields_ = [("schedule", ctypes.c_int32), ("n_prof", ctypes.c_int32), ("prof_n", ctypes.c_void_p),
                ("prof_us", ctypes.c_void_p), ("bytes_full", ctypes.c_double), ("max_chunks", ctypes.c_int32)]


def profile_ops(timeline, steps: int, n: int) -> np.ndarray:
    """Per-chunk cost of every op kind (per step for GATE, COUNTS, K7) from the timeline of
    `steps` fwd+bwd steps run with n chunks: the measure of the union of each kind's event
    intervals per step (launches of one kind that run concurrently -- the push pipeline's fc2 /
    dfc1 on two streams -- count once), divided by n for the chunked kinds (a launch over all
    chunks counts as n chunks' worth)."""
    iv = {}
    for r in timeline:
        k = TIMELINE_TO_OP.get(r["name"])
        if k is not None:
            iv.setdefault(k, []).append((r["start_us"], r["end_us"]))
    tot = np.zeros(N_OPS)
    for k, v in iv.items():
        v.sort()
        s, e, acc = v[0][0], v[0][1], 0.0
        for a, b in v[1:]:
            if a <= e:
                e = max(e, b)
            else:
                acc += e - s
                s, e = a, b
        tot[OPS.index(k)] = acc + (e - s)
    tot /= steps
    for i, k in enumerate(OPS):
        if k not in ONCE:
            tot[i] /= n
    return tot


def tune(profiles: dict, bytes_full: float, schedule: int, max_chunks: int = 8):
    """profiles: {n: profile_ops(...)} for >= 2 chunk counts.  schedule 0: per-chunk launches
    (copy-engine / NCCL paths), 1: push pipeline.  Returns (best_n, pred_us[max_chunks],
    pred_exposed_us[max_chunks])."""
    ns = sorted(profiles)
    prof_n = np.ascontiguousarray(ns, dtype=np.int32)
    prof = np.ascontiguousarray([profiles[n] for n in ns], dtype=np.float64)
    assert prof.shape == (len(ns), N_OPS)
    pred = np.zeros(max_chunks)
    expo = np.zeros(max_chunks)
    best = ctypes.c_int32()
    lib = load_library()
    lib.lancet_tune_chunks.argtypes = [ctypes.POINTER(_TuneInput), ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.POINTER(ctypes.c_int32)]
    lib.lancet_tune_chunks.restype = ctypes.c_int32
    inp = _TuneInput(schedule, len(ns), prof_n.ctypes.data, prof.ctypes.data, float(bytes_full), max_chunks)
    _check(lib.lancet_tune_chunks(ctypes.byref(inp), pred.ctypes.data, expo.ctypes.data, ctypes.byref(best)))
    return best.value, pred, expo
