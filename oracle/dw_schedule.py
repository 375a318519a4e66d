"""Plain CPU oracle of Lancet's weight-gradient computation schedule pass (TEST INFRASTRUCTURE).

Only tests/ may import this module.  It shares no code with the library's native scheduler
(paper_2404_19429_b200/csrc/schedule.cpp) and never imports it.

What it computes (PAPER.md sec:dw_labelling / sec:dw_scheduling, L340-L398, Alg. 1):

  * labelling (L343): "a weight gradient computation instruction I_i can be overlapped with an
    all-to-all instruction I_a if and only if there is no directed path between I_i and I_a"
    -- here from the transitive closure of the dependency graph (Warshall), the plainest
    definition of "path";
  * greedy assignment (Alg. 1 lines 10-21): all-to-alls in program order; for each, while its
    unoverlapped time t_u > 0 and an unused eligible dW exists, take the dW minimising
    |t_u - t_W| (ties -> lowest instruction index), t_u -= t_W;
  * the objective of the integer program (L348-L354): sum_j min(t_a_j, sum_i t_W_i x_ij);
  * an exact assignment by exhaustive enumeration (small instances);
  * the backward program of an L-layer stack of this library's MoE layer (R17), the
    instruction DAG the runtime schedules.
"""
from __future__ import annotations

import itertools

OTHER, A2A, DW = 0, 1, 2


def closure(n: int, edges) -> list[list[bool]]:
    """reach[i][j]: a directed path i -> j of length >= 1 (Warshall's algorithm)."""
    reach = [[False] * n for _ in range(n)]
    for s, t in edges:
        reach[s][t] = True
    for m in range(n):
        for i in range(n):
            if reach[i][m]:
                row_m = reach[m]
                row_i = reach[i]
                for j in range(n):
                    if row_m[j]:
                        row_i[j] = True
    return reach


def label_overlappable(kinds, edges) -> dict[int, list[int]]:
    """W^{I_a} for every all-to-all a (Alg. 1 lines 3-9): the dW instructions
    with no directed path to or from a."""
    n = len(kinds)
    reach = closure(n, edges)
    return {a: [i for i in range(n) if kinds[i] == DW and not reach[i][a] and not reach[a][i]]
            for a in range(n) if kinds[a] == A2A}


def greedy_assign(kinds, cost, sets) -> dict[int, int]:
    """Alg. 1 lines 10-21: returns {dW index: a2a index}."""
    used: set[int] = set()
    asg: dict[int, int] = {}
    for a in range(len(kinds)):
        if kinds[a] != A2A:
            continue
        t_u = cost[a]
        while t_u > 0:
            avail = [i for i in sets[a] if i not in used]
            if not avail:
                break
            j = min(avail, key=lambda i: (abs(t_u - cost[i]), i))
            t_u -= cost[j]
            used.add(j)
            asg[j] = a
    return asg


def objective(kinds, cost, asg) -> float:
    """sum over all-to-alls of min(t_a, sum of the dW time assigned to it)."""
    tot = {a: 0.0 for a in range(len(kinds)) if kinds[a] == A2A}
    for i, a in asg.items():
        tot[a] += cost[i]
    return sum(min(cost[a], s) for a, s in tot.items())


def exact_assign(kinds, cost, sets) -> dict[int, int]:
    """Exhaustive maximiser of the objective under constraints (1)-(2);
    ties -> the lexicographically least choice vector (dW in index order, each choosing an
    a2a index or -1 = unassigned, -1 least).  Guard: <= 12 dW, <= 4 a2a."""
    dws = [i for i in range(len(kinds)) if kinds[i] == DW]
    a2as = [a for a in range(len(kinds)) if kinds[a] == A2A]
    if len(dws) > 12 or len(a2as) > 4:
        raise ValueError("instance too large for the exhaustive oracle")
    options = [[-1] + [a for a in a2as if i in sets[a]] for i in dws]
    best, best_obj = None, -1.0
    for choice in itertools.product(*options):
        asg = {i: a for i, a in zip(dws, choice) if a >= 0}
        ob = objective(kinds, cost, asg)
        if ob > best_obj + 1e-12:
            best, best_obj = asg, ob
    return best


def stack_backward_program(L: int, n: int):
    """Backward instruction DAG of an L-layer stack of MoE layers with n chunks (DESIGN.md
    R17).  Layers are numbered in forward order; the backward runs layer L-1 first.  Per
    layer l, in program order:

        K5[l][c] (combine bwd, c < n), B1[l][c] (a2a #1, dO to the experts),
        DX[l][c] (dX GEMMs), DW2[l], DW1[l] (dW GEMMs over all chunks),
        B2[l][c] (a2a #2, dX back to the token owners), K6[l] (dx gate term), K7[l] (dWg).

    Edges (data dependencies): K5[l][c] -> B1[l][c] -> DX[l][c] -> B2[l][c] -> K6[l];
    B1[l][c] -> DW2[l], DW1[l] (dO received); DX[l][c] -> DW1[l] (dA); K5[l][c] -> K7[l];
    K6[l] -> K5[l-1][c] (dx of layer l is dy of layer l-1).

    Returns (kinds, names, edges, index) with index[(name, l, c)] -> instruction id."""
    kinds, names, edges, index = [], [], [], {}

    def add(kind, name, l, c=0):
        index[(name, l, c)] = len(kinds)
        kinds.append(kind)
        names.append(f"{name}[{l}]" + (f"[{c}]" if name in ("K5", "B1", "DX", "B2") else ""))
        return index[(name, l, c)]

    for l in range(L - 1, -1, -1):
        for c in range(n):
            add(OTHER, "K5", l, c)
        for c in range(n):
            add(A2A, "B1", l, c)
        for c in range(n):
            add(OTHER, "DX", l, c)
        add(DW, "DW2", l)
        add(DW, "DW1", l)
        for c in range(n):
            add(A2A, "B2", l, c)
        add(OTHER, "K6", l)
        add(OTHER, "K7", l)
    for l in range(L):
        for c in range(n):
            edges.append((index[("K5", l, c)], index[("B1", l, c)]))
            edges.append((index[("B1", l, c)], index[("DX", l, c)]))
            edges.append((index[("DX", l, c)], index[("B2", l, c)]))
            edges.append((index[("B2", l, c)], index[("K6", l, 0)]))
            edges.append((index[("B1", l, c)], index[("DW2", l, 0)]))
            edges.append((index[("B1", l, c)], index[("DW1", l, 0)]))
            edges.append((index[("DX", l, c)], index[("DW1", l, 0)]))
            edges.append((index[("K5", l, c)], index[("K7", l, 0)]))
            if l > 0:
                edges.append((index[("K6", l, 0)], index[("K5", l - 1, c)]))
    return kinds, names, edges, index
