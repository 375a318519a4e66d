"""An L-layer stack of MoE layers with Lancet's cross-layer weight-gradient schedule.

PAPER.md Opportunity 1 (L156, Fig. 4b): the dW GEMMs of layer N have no dependency on the
backward all-to-alls of layers N-1, N-2, ..., so they can be moved under them; Alg. 1
(L367-L398) assigns each dW to one all-to-all and the runtime places it "right after" that
all-to-all's launch (L359).  Here every layer is one library context; the assignment comes
from the library's native pass (lancet_stack_dw_plan, R17) and the placement from
its filler slots (LANCET_FLAG_DEFER_DW + lancet_set_dw_fillers), so this module only decides
which context gets which filler list (argument marshalling).  Layers are chained y_l -> x_l+1
(no ops in between), the backward runs L-1 first, dx of layer l is dy of layer l-1.
"""
from __future__ import annotations

from .lancet import FLAG_DEFER_DW, Context, stack_dw_plan

WHICH = (2, 1)          # plan part 0 = dW2 (lancet which bit 1), part 1 = dW1 (bit 0)


class MoEStack:
    def __init__(self, ctxs: list[Context]):
        self.ctxs = ctxs
        self.L = len(ctxs)

    def forward(self, x, params, k, capacity_factor, n_chunks, stream=None):
        """params[l] = (wg, w1, w2).  Returns the per-layer outputs [y_0 .. y_L-1]."""
        ys = []
        for ctx, (wg, w1, w2) in zip(self.ctxs, params):
            y, _, _, _ = ctx.forward(x, wg, w1, w2, k, capacity_factor, n_chunks, stream=stream,
                                     routing=False)
            ys.append(y)
            x = y
        self.n = n_chunks
        return ys

    def backward(self, dy, grads, plan=None, stream=None):
        """grads[l] = (dwg, dw1, dw2) output buffers.  plan = (host_layer, host_a2a) from
        `plan_from_costs` (or hand-made), None = every layer keeps its own dW schedule.
        Returns the per-layer dx [dx_0 .. dx_L-1] (dx_0 is the stack's input gradient)."""
        L, n = self.L, self.n
        fill = [[] for _ in range(L)]
        defer = [False] * L
        if plan is not None:
            hl, ha = plan
            for m in range(L):
                if hl[m][0] < 0 and hl[m][1] < 0:
                    continue
                defer[m] = True
                for w in range(2):
                    if hl[m][w] >= 0:
                        assert hl[m][w] <= m, "a dW can only move to a later backward"
                        fill[hl[m][w]].append((self.ctxs[m], WHICH[w], int(ha[m][w])))
                    else:              # unassigned part keeps its place: after its own dX GEMMs
                        fill[m].append((self.ctxs[m], WHICH[w], n))
        dxs = [None] * L
        base = [c.cfg.flags & ~FLAG_DEFER_DW for c in self.ctxs]
        for l in range(L - 1, -1, -1):
            ctx = self.ctxs[l]
            ctx.set_flags(base[l] | (FLAG_DEFER_DW if defer[l] else 0))
            ctx.set_dw_fillers(fill[l])
            dwg, dw1, dw2 = grads[l]
            dx, _, _, _ = ctx.backward(dy, dwg=dwg, dw1=dw1, dw2=dw2, stream=stream)
            dxs[l] = dx
            dy = dx
        for l in range(L):
            self.ctxs[l].set_flags(base[l])
        return dxs


def plan_from_costs(t_a2a, t_dw):
    """Alg. 1 over the stack (native pass).  t_a2a [L][2n] us per all-to-all in issue order,
    t_dw [L][2] us of (dW2, dW1) -- e.g. measured from a timeline of the default schedule."""
    return stack_dw_plan(t_a2a, t_dw)


def costs_from_timelines(timelines, n):
    """Per-op costs for the plan from one timeline per layer (lancet timeline records of a
    step under the default schedule): mean event-span time of each all-to-all in issue order
    (a2a_bwd_dispatch chunk c -> c, a2a_bwd_combine chunk c -> n + c) and of the dW GEMMs."""
    import numpy as np
    L = len(timelines)
    t_a2a = np.zeros((L, 2 * n))
    t_dw = np.zeros((L, 2))
    for l, tl in enumerate(timelines):
        cnt_a = np.zeros(2 * n)
        for r in tl:
            dur = r["end_us"] - r["start_us"]
            c = max(r["chunk"], 0)
            if r["name"] == "a2a_bwd_dispatch":
                t_a2a[l, c] += dur; cnt_a[c] += 1
            elif r["name"] == "a2a_bwd_combine":
                t_a2a[l, n + c] += dur; cnt_a[n + c] += 1
            elif r["name"] == "expert_dw2":
                t_dw[l, 0] += dur
            elif r["name"] == "expert_dw1":
                t_dw[l, 1] += dur
        steps = max(1, int(cnt_a.max()))
        t_a2a[l] /= np.maximum(cnt_a, 1)
        t_dw[l] /= steps
    return t_a2a, t_dw
