"""Chunk-count tuner for the pipelined MoE layer.

Lancet picks the number of partitions with a dynamic program over partition ranges whose
objective is the time a stage simulator predicts from profiled operator costs (PAPER.md
P:L413, "T(n)"; the simulator P:L494-L499 runs the stages on a computation and a
communication lane in their issue order).  For one MoE layer there is a single partition
range, so the DP reduces to a scan over n: this module simulates the S1/S2 schedule of
lancet.cu (the same ops, lanes, issue order and dependencies) for each candidate n with
per-op costs fitted from measured timelines, and returns the n with the smallest predicted
step time.

Cost model per op type (fitted by `fit` from bench.py lines measured at two chunk counts):
a chunked op's per-chunk duration is  fixed + whole / n  (launch / protocol latency plus its
share of the work); once-per-step ops (gate, permute, counts exchange) are constants.
"""
from __future__ import annotations

from dataclasses import dataclass, field

CHUNKED = ("a2a_dispatch", "a2a_combine", "a2a_bwd_dispatch", "a2a_bwd_combine", "expert_fc1",
           "expert_fc2", "expert_dfc2", "expert_dfc1", "expert_dw2", "expert_dw1", "combine",
           "combine_bwd", "unpermute_gate_bwd")
ONCE = ("gate", "permute", "a2a_counts", "gate_dwg")


@dataclass
class OpModel:
    fixed: float = 0.0   # us per chunk launch
    whole: float = 0.0   # us of the whole batch's work

    def per_chunk(self, n: int) -> float:
        return self.fixed + self.whole / n


@dataclass
class CostModel:
    chunked: dict = field(default_factory=dict)   # name -> OpModel
    once: dict = field(default_factory=dict)      # name -> us

    def t(self, name: str, n: int) -> float:
        if name in self.chunked:
            return self.chunked[name].per_chunk(n)
        return self.once.get(name, 0.0)


def fit(lines: dict) -> CostModel:
    """lines: {n: bench.py JSON} for two (or more) chunk counts, measured on the expert-parallel
    path.  Per chunked op: per-chunk time t_n = us_per_step / groups_per_step; least squares of
    t_n = fixed + whole / n over the given n."""
    m = CostModel()
    ns = sorted(lines)
    for name in CHUNKED:
        pts = []
        for n in ns:
            k = lines[n]["kernels"].get(name)
            groups = lines[n].get("launch_groups", {}).get(name)
            if k is None:
                continue
            g = groups or n
            pts.append((1.0 / n, k["us"] / g))
        if not pts:
            continue
        if len(pts) == 1:
            m.chunked[name] = OpModel(0.0, pts[0][1] / pts[0][0])
            continue
        xs = [p[0] for p in pts]
        ys = [p[1] for p in pts]
        xm, ym = sum(xs) / len(xs), sum(ys) / len(ys)
        sxx = sum((x - xm) ** 2 for x in xs)
        b = sum((x - xm) * (y - ym) for x, y in zip(xs, ys)) / sxx if sxx > 0 else ym / xm
        a = ym - b * xm
        m.chunked[name] = OpModel(max(0.0, a), max(0.0, b))
    for name in ONCE:
        vals = [lines[n]["kernels"][name]["us"] for n in ns if name in lines[n]["kernels"]]
        if vals:
            m.once[name] = sum(vals) / len(vals)
    return m


def simulate(m: CostModel, n: int, dw_overlap: bool = True, serial: bool = False) -> dict:
    """Two-lane in-order simulation of one forward + backward of lancet.cu's expert-parallel
    schedule with n chunks (serial: one lane, LANCET_FLAG_SERIAL's unoverlapped baseline).
    Returns the predicted step time and exposed communication (us)."""
    lanes = {"comp": 0.0, "comm": 0.0}
    done = {}
    busy = {"comp": [], "comm": []}

    def run(name, lane, deps=(), after=0.0, chunk=None):
        kind = lane                      # exposure is judged by op kind, whatever lane runs it
        if serial:
            lane = "comp"
        key = name if chunk is None else (name, chunk)
        start = max([lanes[lane], after] + [done[d] for d in deps])
        end = start + m.t(name, n)
        lanes[lane] = end
        done[key] = end
        busy[kind].append((start, end))
        return key

    # ---- forward (S1): gate, counts exchange (host waits for it), permute, D0..Dn-1,
    #      experts per chunk, C0..Cn-1, gathers per chunk
    g = run("gate", "comp")
    cnt = run("a2a_counts", "comm", deps=[g])
    p = run("permute", "comp", deps=[g])
    host = done[cnt]                     # the one host synchronisation of the step
    disp = [run("a2a_dispatch", "comm", deps=[p, cnt], chunk=c) for c in range(n)]
    exp = []
    for c in range(n):
        a = run("expert_fc1", "comp", deps=[disp[c]], after=host, chunk=c)
        exp.append(run("expert_fc2", "comp", deps=[a], chunk=c))
    comb = [run("a2a_combine", "comm", deps=[exp[c]], chunk=c) for c in range(n)]
    for c in range(n):
        run("combine", "comp", deps=[comb[c]], chunk=c)
    # ---- backward (S2): K5 per chunk, b1 per chunk, dX then dW per chunk, b2, K6 per chunk, K7
    k5 = [run("combine_bwd", "comp", chunk=c) for c in range(n)]
    b1 = [run("a2a_bwd_dispatch", "comm", deps=[k5[c]], chunk=c) for c in range(n)]
    dx = []
    for c in range(n):
        a = run("expert_dfc2", "comp", deps=[b1[c]], chunk=c)
        dx.append(run("expert_dfc1", "comp", deps=[a], chunk=c))
        if dw_overlap:
            w = run("expert_dw2", "comp", deps=[dx[c]], chunk=c)
            run("expert_dw1", "comp", deps=[w], chunk=c)
    b2 = [run("a2a_bwd_combine", "comm", deps=[dx[c]], chunk=c) for c in range(n)]
    if not dw_overlap:
        for c in range(n):
            w = run("expert_dw2", "comp", chunk=c)
            run("expert_dw1", "comp", deps=[w], chunk=c)
    for c in range(n):
        run("unpermute_gate_bwd", "comp", deps=[b2[c]], chunk=c)
    run("gate_dwg", "comp")
    step = max(lanes.values())

    def union(iv):
        out = []
        for a, b in sorted(iv):
            if out and a <= out[-1][1]:
                out[-1][1] = max(out[-1][1], b)
            else:
                out.append([a, b])
        return out
    comm, comp = union(busy["comm"]), union(busy["comp"])
    cover = sum(max(0.0, min(b, d) - max(a, c)) for a, b in comm for c, d in comp)
    return {"n": n, "step_us": step, "exposed_comm_us": sum(b - a for a, b in comm) - cover,
            "comm_us": sum(b - a for a, b in comm)}


def best_n(m: CostModel, candidates=(1, 2, 4, 8)) -> tuple[int, list]:
    preds = [simulate(m, n) for n in candidates]
    return min(preds, key=lambda p: p["step_us"])["n"], preds
