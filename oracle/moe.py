"""Plain CPU oracle of Lancet's expert-parallel MoE layer step (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference) may
import this module.  It shares no code with paper_2404_19429_b200/ (the CUDA path) and
never imports it; both read inputs from synthetic/.

What it computes.  Lancet's partitioning "maintain[s] mathematical equivalence" (PAPER.md
L88) and capacity passing preserves "the exact token-to-expert mapping and token dropping
as the un-partitioned case" (L256).  So the oracle is the plain, UNPARTITIONED MoE layer
(L108-L119, L123, L245-L248) over G simulated ranks, written step by step:

  gate (L123) -> top-k (L123) -> capacity C per (rank, expert) (L118-L119) -> token-major
  admission (R7/R8) -> expert FFN (L62, L108) -> gather/combine (L62, L248);
  backward by the chain rule (formulas in DESIGN.md "Backward"; pinned by finite
  differences in tests/test_oracle_backward.py).

Floating point: fp64 everywhere except the gate logits, which follow the fp32 fma chain of
DESIGN.md R1 (oracle/gate_logits.c) so that routing can be compared bit for bit.
Matrix products use numpy's fp64 matmul as a library primitive.

Parity status: every function here is pinned by a CPU test;
numeric MoE outputs are pinned by definitions and invariants, not by paper-printed values
(the paper prints none beyond the 3/4C-1/4C example, L253-L256).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native

DROPPED = -1
ACTS = ("gelu_tanh", "relu", "identity_expert")


# ----------------------------------------------------------------------------------------
# Routing
# ----------------------------------------------------------------------------------------

def capacity(T: int, k: int, E: int, cf: float) -> int:
    """Expert capacity C per (source rank, expert).

    "restrict the maximum tokens assigned to each expert (expert capacity, C) on each
    device".  Formula and rounding are DESIGN.md reading R4:
    C = max(1, min(T, ceil(cf*k*T/E))), evaluated in double, T = the rank's whole batch.
    """
    return max(1, min(T, math.ceil(cf * k * T / E)))


def gate_logits(x: np.ndarray, wg: np.ndarray) -> np.ndarray:
    """logit = x @ Wg as the fp32 fma chain of DESIGN.md R1 ("a gating score for each
    expert using a trainable linear layer").  [T,d] x [d,E] -> [T,E] f32."""
    return _native.gate_logits(x, wg)


def topk(logits: np.ndarray, k: int) -> np.ndarray:
    """"choosing k experts with highest scores (top-k routing)".

    Selection key (R2): logit descending, ties to the lower expert index.  A
    stable sort of -logit keeps equal keys in index order.  Returns idx [T,k] int32 in rank
    order (idx[:,0] is the best expert)."""
    order = np.argsort(-logits, axis=1, kind="stable")
    return order[:, :k].astype(np.int32)


def softmax(logits: np.ndarray) -> np.ndarray:
    """p[t,e] = exp(logit - max) / sum_e exp(logit - max), in fp64 (R3)."""
    l64 = logits.astype(np.float64)
    z = np.exp(l64 - l64.max(axis=1, keepdims=True))
    return z / z.sum(axis=1, keepdims=True)


def combine_weights(p: np.ndarray, idx: np.ndarray, renormalize: bool = False) -> np.ndarray:
    """w[t,j] = p[t, idx[t,j]] (Switch convention, R3); with `renormalize`, divided
    by the sum over the k selected experts.  Normalisation happens before any drop."""
    w = np.take_along_axis(p, idx.astype(np.int64), axis=1)
    if renormalize:
        w = w / w.sum(axis=1, keepdims=True)
    return w


def assign_slots(idx: np.ndarray, E: int, C: int, used=None):
    """Capacity admission in token-major order (R7, R8).

    Scan the flattened (t, j) pairs in lexicographic order; expert e admits a pair while it
    has fewer than C tokens ("Any excess tokens assigned to an expert are discarded",
    PAPER.md L119).  slot = the pair's position in e's buffer, DROPPED (-1) otherwise.
    `used` is the carried capacity state (per-expert admitted count) -- the "capacity
    information" passed between partitions; returns (slot, used)."""
    T, k = idx.shape
    used = [0] * E if used is None else list(used)
    slot = np.full((T, k), DROPPED, dtype=np.int32)
    for t in range(T):
        for j in range(k):
            e = int(idx[t, j])
            if used[e] < C:
                slot[t, j] = used[e]
                used[e] += 1
    return slot, used


def importance_scores(logits: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """Batch Prioritized Routing's importance score: "the sum of top-k largest gating
    scores".  Gating score = the softmax probability p (R3), so
    s_t = sum_j p[t, idx[t,j]], evaluated in fp64 as

        s_t = (sum_j exp(l[t, idx_j] - m_t)) / (sum_e exp(l[t, e] - m_t)),  m_t = max_e l[t, e],

    both sums sequential (j in rank order, e ascending) -- DESIGN.md R16.  The score decides
    integers (who is dropped), so both sides evaluate it in fp64 in this order."""
    l64 = logits.astype(np.float64)
    T, E = l64.shape
    m = l64.max(axis=1)
    Z = np.zeros(T)
    for e in range(E):
        Z = Z + np.exp(l64[:, e] - m)
    num = np.zeros(T)
    for j in range(idx.shape[1]):
        num = num + np.exp(l64[np.arange(T), idx[:, j]] - m)
    return num / Z


def assign_slots_bpr(idx: np.ndarray, score: np.ndarray, E: int, C: int):
    """Batch Prioritized Routing (riquelme2021bpr) in Lancet's
    partition-after-gate mode (L270-L271, fig:part_after_gate): the router "sorts tokens in a
    batch first by their importance score ... and then assigns tokens to experts. So tokens
    with lower scores would be dropped first."  Step by step (R16):

      1. order the tokens by (score descending, token index ascending);
      2. walk the tokens in that order, each token's choices j in rank order; expert e admits
         a pair while it holds fewer than C ("any excess tokens ... are discarded", L119);
      3. slot = the pair's position among e's ADMITTED pairs in token-major order (R7/R8), so
         that chunk c's rows of e stay one contiguous slot range (the partition happens
         after the gate; capacity passing is again the prefix at chunk boundaries).

    Returns slot [T,k] int32 (-1 dropped)."""
    T, k = idx.shape
    order = sorted(range(T), key=lambda t: (-score[t], t))
    used = [0] * E
    admitted = np.zeros((T, k), dtype=bool)
    for t in order:
        for j in range(k):
            e = int(idx[t, j])
            if used[e] < C:
                admitted[t, j] = True
                used[e] += 1
    slot = np.full((T, k), DROPPED, dtype=np.int32)
    nxt = [0] * E
    for t in range(T):
        for j in range(k):
            if admitted[t, j]:
                e = int(idx[t, j])
                slot[t, j] = nxt[e]
                nxt[e] += 1
    return slot


def route_micro_bpr(idx: np.ndarray, score: np.ndarray, E: int, C: int, n_chunks: int):
    """BPR applied per micro-batch with capacity passing -- what partitioning BEFORE the gate
    would do (diagnostic only).  PAPER.md L270: "Splitting along batch dimension would thus
    cause differences in token dropping" -- the reason BPR only allows partitioning after the
    MoE gate.  Chunk c sorts only its own tokens and gets the capacity chunks 0..c-1 left."""
    bounds = chunk_bounds(idx.shape[0], n_chunks)
    used = [0] * E
    admitted = np.zeros(idx.shape, dtype=bool)
    for c in range(n_chunks):
        for t in sorted(range(bounds[c], bounds[c + 1]), key=lambda t: (-score[t], t)):
            for j in range(idx.shape[1]):
                e = int(idx[t, j])
                if used[e] < C:
                    admitted[t, j] = True
                    used[e] += 1
    return admitted


_GOLDEN_GAMMA = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


def splitmix64(key: int, seed: int) -> int:
    """SplitMix64 output for counter `key` (0-based) of the stream seeded with `seed`: the
    state after key + 1 increments of the golden-gamma Weyl sequence, through the SplitMix64
    finaliser (Steele, Lea and Flood 2014).  DESIGN.md R18."""
    z = (seed + (key + 1) * _GOLDEN_GAMMA) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def random_gate(T: int, E: int, k: int, seed: int):
    """Random gating ("Random [zuo2022taming, chen2023sparse] gating", whose
    "expert assignment can be decided from partial batches"), R18: token t's j-th
    expert is the r-th smallest expert not chosen by draws 0..j-1, r = splitmix64(8 t + j,
    seed) mod (E - j) (distinct experts, uniform up to a < 2^-50 modulo bias); combine weights
    1/k.  The draw depends on the token index only, so any partition reproduces it.
    Returns idx [T,k] int32 and w [T,k] f64."""
    idx = np.zeros((T, k), dtype=np.int32)
    for t in range(T):
        free = list(range(E))
        for j in range(k):
            r = splitmix64(8 * t + j, seed) % (E - j)
            idx[t, j] = free.pop(r)
    return idx, np.full((T, k), 1.0 / k)


def chunk_bounds(T: int, n: int) -> list[int]:
    """Split T tokens into n contiguous chunks whose sizes differ by at most one, larger
    first (R9).  Returns the n+1 boundaries [t_0=0, ..., t_n=T]."""
    assert 1 <= n <= max(T, 1)
    base, extra = divmod(T, n)
    b = [0]
    for c in range(n):
        b.append(b[-1] + base + (1 if c < extra else 0))
    return b


def route_micro(idx: np.ndarray, E: int, C: int, n_chunks: int):
    """Partitioned gating with capacity passing (fig:proposed_partition):
    chunk c is admitted with the capacity left over by chunks 0..c-1.  Returns the
    concatenated slots and the per-chunk admitted counts n[e][c]."""
    bounds = chunk_bounds(idx.shape[0], n_chunks)
    used = [0] * E
    slots, counts = [], np.zeros((E, n_chunks), dtype=np.int64)
    for c in range(n_chunks):
        before = list(used)
        s, used = assign_slots(idx[bounds[c]:bounds[c + 1]], E, C, used)
        slots.append(s)
        for e in range(E):
            counts[e, c] = used[e] - before[e]
    return np.concatenate(slots, axis=0), counts


def route_micro_naive(idx: np.ndarray, E: int, C_chunk: int, n_chunks: int):
    """Direct micro-batching WITHOUT capacity passing: each chunk gets its own capacity
    C_chunk ("each processed with expert capacity 1/2 C").  Diagnostic only
    -- it is the behaviour Lancet avoids."""
    bounds = chunk_bounds(idx.shape[0], n_chunks)
    return np.concatenate([assign_slots(idx[bounds[c]:bounds[c + 1]], E, C_chunk)[0]
                           for c in range(n_chunks)], axis=0)


def chunk_counts(idx: np.ndarray, slot: np.ndarray, E: int, n_chunks: int) -> np.ndarray:
    """Admitted rows per (expert, chunk): n[e][c] = #{(t,j): t in chunk c, idx=e, slot>=0}."""
    bounds = chunk_bounds(idx.shape[0], n_chunks)
    counts = np.zeros((E, n_chunks), dtype=np.int64)
    for c in range(n_chunks):
        i, s = idx[bounds[c]:bounds[c + 1]], slot[bounds[c]:bounds[c + 1]]
        for e in range(E):
            counts[e, c] = int(np.count_nonzero((i == e) & (s >= 0)))
    return counts


def size_matrix(send_counts: list[np.ndarray], G: int) -> np.ndarray:
    """The sizes exchanged by the first all-to-all of fig:irregular_implementations
    (PAPER.md L517, L525): N[src][dst][c] = rows rank src sends to rank dst in chunk c,
    where expert e lives on rank e // E_l (contiguous placement, G = E / E_l)."""
    E, n = send_counts[0].shape
    E_l = E // G
    N = np.zeros((G, G, n), dtype=np.int64)
    for src in range(G):
        for e in range(E):
            N[src, e // E_l] += send_counts[src][e]
    return N


def recv_counts(send_counts: list[np.ndarray], G: int, rank: int) -> np.ndarray:
    """Rows rank `rank` receives: R[src][e_l][c] = send_counts[src][rank*E_l + e_l][c]."""
    E, n = send_counts[0].shape
    E_l = E // G
    return np.stack([send_counts[src][rank * E_l:(rank + 1) * E_l] for src in range(G)])


# ----------------------------------------------------------------------------------------
# Expert FFN
# ----------------------------------------------------------------------------------------

_GELU_C = math.sqrt(2.0 / math.pi)


def act_fwd(a: np.ndarray, act: str) -> np.ndarray:
    """Expert activation (R5): GPT-2's gelu_new (tanh form) by default."""
    if act == "gelu_tanh":
        return 0.5 * a * (1.0 + np.tanh(_GELU_C * (a + 0.044715 * a ** 3)))
    if act == "relu":
        return np.maximum(a, 0.0)
    raise ValueError(act)


def act_grad(a: np.ndarray, act: str) -> np.ndarray:
    """d act / d a."""
    if act == "gelu_tanh":
        u = _GELU_C * (a + 0.044715 * a ** 3)
        th = np.tanh(u)
        return 0.5 * (1.0 + th) + 0.5 * a * (1.0 - th * th) * _GELU_C * (1.0 + 3 * 0.044715 * a * a)
    if act == "relu":
        return (a > 0).astype(np.float64)
    raise ValueError(act)


def expert_ffn(x: np.ndarray, w1: np.ndarray, w2: np.ndarray, act: str):
    """One expert ("Each expert processes the C received tokens"; an FFN,
    L108): a = x W1^T, h = act(a), o = h W2^T, no biases (R5).  x [M,d], W1 [f,d], W2 [d,f]."""
    a = x.astype(np.float64) @ w1.astype(np.float64).T
    h = act_fwd(a, act)
    o = h @ w2.astype(np.float64).T
    return a, h, o


# ----------------------------------------------------------------------------------------
# The layer over G simulated ranks
# ----------------------------------------------------------------------------------------

@dataclass
class RankRouting:
    logits: np.ndarray     # [T,E] f32 (f64 with gate_fp64)
    idx: np.ndarray        # [T,k] i32
    p: np.ndarray          # [T,E] f64
    w: np.ndarray          # [T,k] f64
    slot: np.ndarray       # [T,k] i32 (-1 dropped)
    C: int
    counts: np.ndarray     # [E,n] admitted rows per expert per chunk
    gate: str = "switch"   # "switch" | "bpr" | "random"


@dataclass
class LayerResult:
    routing: list                          # RankRouting per rank
    y: list                                # [T,d] f64 per rank
    saved: dict = field(default_factory=dict)   # (rank, expert) -> (t, j, a, h, o)


def route_rank(x, wg, k, cf, n_chunks, renormalize=False, gate_fp64=False,
               gate="switch", seed=0) -> RankRouting:
    """Routing of one rank's local batch (routing never crosses ranks: the gate is
    replicated, and C is per device).  `gate_fp64` replaces the R1 fp32
    chain by an fp64 product -- used only by the finite-difference pins of the backward,
    which need a gate that is smooth at the 1e-6 scale.  `gate`: "switch" (token-major
    admission, R7) or "bpr" (Batch Prioritized Routing, assign_slots_bpr, R16)."""
    T = x.shape[0]
    E = wg.shape[1]
    if gate == "random":
        # no gate network: logits are reported as zeros, and no gradient reaches Wg (R18)
        idx, w = random_gate(T, E, k, seed)
        C = capacity(T, k, E, cf)
        slot, _ = assign_slots(idx, E, C)
        return RankRouting(np.zeros((T, E), np.float32), idx, np.zeros((T, E)), w, slot, C,
                           chunk_counts(idx, slot, E, n_chunks), gate="random")
    if gate_fp64:
        logits = x.astype(np.float64) @ wg.astype(np.float64)
    else:
        logits = gate_logits(x, wg)
    idx = topk(logits, k)
    p = softmax(logits)
    w = combine_weights(p, idx, renormalize)
    C = capacity(T, k, E, cf)
    if gate == "bpr":
        slot = assign_slots_bpr(idx, importance_scores(logits, idx), E, C)
    elif gate == "switch":
        slot, _ = assign_slots(idx, E, C)
    else:
        raise ValueError(gate)
    counts = chunk_counts(idx, slot, E, n_chunks)
    return RankRouting(logits, idx, p, w, slot, C, counts, gate=gate)


def expert_weights(w1_ranks, w2_ranks, e, E_l):
    """Weights of global expert e, which lives on rank e // E_l (P:L517 G = E / E_l)."""
    return w1_ranks[e // E_l][e % E_l], w2_ranks[e // E_l][e % E_l]


def forward(xs, wg, w1_ranks, w2_ranks, k, cf, n_chunks, act="gelu_tanh",
            renormalize=False, token_subset=None, gate_fp64=False, gate="switch",
            seed=0, experts=None) -> LayerResult:
    """The MoE layer forward over G = len(xs) ranks.

    xs[r]: [T_r, d] tokens of rank r; w1_ranks[r]: [E_l, f, d], w2_ranks[r]: [E_l, d, f].
    Output y_t = sum over admitted choices j of w[t,j] * FFN_{idx[t,j]}(x_t)  (gather
    "restores the received tokens back to their original order"; dropped choices
    contribute zero, R6).  `token_subset` (list per rank of token ids, or None) restricts
    the expert math to those tokens (routing is always over the whole batch); y rows of
    other tokens are NaN.  `experts` (global expert ids, or None) restricts the expert math
    to those experts -- a cost restriction for large shapes: y then holds only their
    contributions, and backward() gives the full dW1 / dW2 of exactly those experts.

    The all-to-all is pure data movement: a token's expert output depends only
    on the token and the expert's weights, so the oracle evaluates each expert on the rows
    admitted to it directly; saved[(r, e)] keeps (t, j, a, h, o) for the backward."""
    G = len(xs)
    E = wg.shape[1]
    E_l = E // G
    res = LayerResult(routing=[], y=[])
    for r in range(G):
        rt = route_rank(xs[r], wg, k, cf, n_chunks, renormalize, gate_fp64, gate, seed)
        res.routing.append(rt)
        T, d = xs[r].shape
        keep = np.zeros(T, dtype=bool)
        keep[np.arange(T) if token_subset is None else np.asarray(token_subset[r], dtype=np.int64)] = True
        y = np.full((T, d), np.nan)
        y[keep] = 0.0
        for e in (range(E) if experts is None else sorted(set(experts))):
            # admitted pairs of expert e, in token-major (buffer slot) order
            t_sel, j_sel = np.nonzero((rt.idx == e) & (rt.slot >= 0) & keep[:, None])
            if t_sel.size == 0:
                continue
            xe = xs[r][t_sel].astype(np.float64)
            if act == "identity_expert":
                a = h = None
                o = xe
            else:
                w1e, w2e = expert_weights(w1_ranks, w2_ranks, e, E_l)
                a, h, o = expert_ffn(xe, w1e, w2e, act)
            np.add.at(y, t_sel, rt.w[t_sel, j_sel][:, None] * o)
            res.saved[(r, e)] = (t_sel, j_sel, a, h, o)
        res.y.append(y)
    return res


def backward(fwd: LayerResult, xs, wg, w1_ranks, w2_ranks, dys, act="gelu_tanh",
             renormalize=False):
    """Gradients of sum_r <dy_r, y_r> by the chain rule:

      g[t,j]   = <dy_t, o_tj>           (admitted; 0 for dropped choices)
      dout_tj  = w[t,j] dy_t;  dh = dout W2_e;  da = dh * act'(a)
      dW2_e   += dout^T h;     dW1_e += da^T x_t;   dx_t += da W1_e
      dlogit   = p * (g~ - sum_j g_j w_j)              (no renormalisation; g~_e = g_j at
                                                         e = idx_j, else 0)
               = q_j (g_j - sum_j' g_j' q_j') at idx  (renormalised, q = w), 0 elsewhere
      dx_t    += dlogit_t Wg^T;  dWg_r = x_r^T dlogit_r (per rank; the DP all-reduce of
                 the replicated gate, is the caller's).
    Top-k and capacity decisions are piecewise constant and carry no gradient.
    Returns dict(dx=[per rank], dwg=[per rank], g=[per rank], dlogit=[per rank],
    and unless identity experts dw1=[per rank [E_l,f,d]], dw2=[per rank [E_l,d,f]])."""
    G = len(xs)
    E = wg.shape[1]
    E_l = E // G
    d = xs[0].shape[1]
    ident = act == "identity_expert"
    if not ident:
        f = w1_ranks[0].shape[1]
        dw1 = [np.zeros((E_l, f, d)) for _ in range(G)]
        dw2 = [np.zeros((E_l, d, f)) for _ in range(G)]
    dxs, dwgs, gs, dlogits = [], [], [], []
    wg64 = wg.astype(np.float64)
    for r in range(G):
        rt = fwd.routing[r]
        x = xs[r].astype(np.float64)
        dy = dys[r].astype(np.float64)
        T, k = rt.idx.shape
        dx = np.zeros((T, d))
        g = np.zeros((T, k))
        for e in range(E):
            if (r, e) not in fwd.saved:
                continue
            t_sel, j_sel, a, h, o = fwd.saved[(r, e)]
            g[t_sel, j_sel] = np.sum(dy[t_sel] * o, axis=1)
            dout = rt.w[t_sel, j_sel][:, None] * dy[t_sel]
            if ident:
                np.add.at(dx, t_sel, dout)
                continue
            w1e, w2e = expert_weights(w1_ranks, w2_ranks, e, E_l)
            dh = dout @ w2e.astype(np.float64)
            da = dh * act_grad(a, act)
            dw2[e // E_l][e % E_l] += dout.T @ h
            dw1[e // E_l][e % E_l] += da.T @ x[t_sel]
            np.add.at(dx, t_sel, da @ w1e.astype(np.float64))
        dlogit = np.zeros((T, E))
        s = np.sum(g * rt.w, axis=1)                       # sum_j g_j w_j
        if rt.gate == "random":
            pass                                           # no gate network (R18)
        elif renormalize:
            for j in range(k):
                dlogit[np.arange(T), rt.idx[:, j]] = rt.w[:, j] * (g[:, j] - s)
        else:
            gt = np.zeros((T, E))
            for j in range(k):
                gt[np.arange(T), rt.idx[:, j]] = g[:, j]
            dlogit = rt.p * (gt - s[:, None])
        dx += dlogit @ wg64.T
        dxs.append(dx)
        dwgs.append(x.T @ dlogit)
        gs.append(g)
        dlogits.append(dlogit)
    out = dict(dx=dxs, dwg=dwgs, g=gs, dlogit=dlogits)
    if not ident:
        out.update(dw1=dw1, dw2=dw2)
    return out
