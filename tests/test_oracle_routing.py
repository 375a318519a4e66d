"""Pins of the oracle's routing (gate logits, top-k, softmax, capacity, slots, chunks, sizes)
against things other than itself: closed forms, brute force, the paper's worked example,
SPEC.md's hand examples, a hand-derived golden fixture and invariants."""
import itertools
import json
import math
import os

import numpy as np
import pytest
import scipy.special

import synthetic as S
from oracle import moe

rng = np.random.default_rng(1234)


# ---------------------------------------------------------------- gate logits (R1) ----

def test_gate_logits_one_hot_rows_select_wg_rows():
    d, E = 7, 5
    wg = rng.standard_normal((d, E)).astype(np.float32)
    x = np.eye(d, dtype=np.float32)
    assert np.array_equal(moe.gate_logits(x, wg), wg)          # logit[t] = Wg[t,:] exactly


def test_gate_logits_exact_for_small_integers():
    # all products and partial sums exactly representable -> any correct order is exact
    x = rng.integers(-8, 9, size=(33, 19)).astype(np.float32)
    wg = rng.integers(-8, 9, size=(19, 6)).astype(np.float32)
    want = x.astype(np.int64) @ wg.astype(np.int64)
    assert np.array_equal(moe.gate_logits(x, wg), want.astype(np.float32))


def test_gate_logits_within_fp32_dot_error_bound():
    # |fl(sum) - sum| <= gamma_d * sum|x_i w_i|, gamma_d = d u / (1 - d u), u = 2^-24
    x = S.gen_tokens(3, 0, 64, 256)
    wg = S.gen_gate(3, 256, 8, 0.5)
    got = moe.gate_logits(x, wg).astype(np.float64)
    exact = x.astype(np.float64) @ wg.astype(np.float64)
    u = 2.0 ** -24
    gamma = 256 * u / (1 - 256 * u)
    bound = gamma * (np.abs(x.astype(np.float64)) @ np.abs(wg.astype(np.float64)))
    assert np.all(np.abs(got - exact) <= bound)
    # a transposed / mis-indexed Wg would be far outside the bound
    assert np.max(np.abs(got - exact)) < 1e-4 * np.max(np.abs(exact))


def test_gate_logits_chain_is_fused_and_in_increasing_i():
    # fused: round(x1*w1 + acc) once.  x1*w1 = 1 + 2^-11 + 2^-24; unfused rounding of the
    # product loses the 2^-24 (tie to even), fused keeps it.
    a = np.float32(1 + 2.0 ** -12)
    x = np.array([[-1.0, a]], dtype=np.float32)
    wg = np.array([[1.0], [a]], dtype=np.float32)
    assert moe.gate_logits(x, wg)[0, 0] == np.float32(2.0 ** -11 + 2.0 ** -24)
    # order: 1 + 2^-24 + 2^-24 in increasing i rounds to 1 twice; any other order gives 1+2^-23
    x = np.array([[1.0, 2.0 ** -24, 2.0 ** -24]], dtype=np.float32)
    wg = np.ones((3, 1), dtype=np.float32)
    assert moe.gate_logits(x, wg)[0, 0] == np.float32(1.0)


# ---------------------------------------------------------------- top-k (R2) ----------

def _brute_rank_topk(logits, k):
    """rank(e) = #experts strictly better under (logit desc, index asc); idx[j] = rank j."""
    T, E = logits.shape
    out = np.empty((T, k), dtype=np.int32)
    for t in range(T):
        for e in range(E):
            r = sum(1 for e2 in range(E)
                    if logits[t, e2] > logits[t, e] or (logits[t, e2] == logits[t, e] and e2 < e))
            if r < k:
                out[t, r] = e
    return out


@pytest.mark.parametrize("E,k", [(4, 1), (4, 2), (8, 2), (8, 3), (16, 4)])
def test_topk_matches_rank_brute_force_with_ties(E, k):
    logits = rng.integers(-3, 4, size=(200, E)).astype(np.float32)   # many ties
    assert np.array_equal(moe.topk(logits, k), _brute_rank_topk(logits, k))


def test_topk_best_subset_by_enumeration():
    # the chosen set maximises the sum of logits over all k-subsets (distinct logits)
    logits = rng.standard_normal((50, 6)).astype(np.float32)
    idx = moe.topk(logits, 3)
    for t in range(50):
        best = max(itertools.combinations(range(6), 3), key=lambda s: sum(logits[t, list(s)]))
        assert set(idx[t]) == set(best)


def test_topk_signed_zero_is_a_tie():
    logits = np.array([[-0.0, 0.0, -1.0]], dtype=np.float32)
    assert moe.topk(logits, 2).tolist() == [[0, 1]]


# ---------------------------------------------------------------- softmax / weights ----

def test_softmax_matches_scipy_and_is_shift_invariant():
    l = (rng.standard_normal((40, 8)) * 5).astype(np.float32)
    p = moe.softmax(l)
    assert np.allclose(p, scipy.special.softmax(l.astype(np.float64), axis=1), rtol=1e-13, atol=0)
    assert np.allclose(p.sum(1), 1.0, rtol=1e-14)
    assert np.allclose(moe.softmax(l + np.float32(3.0)), p, rtol=1e-6)


def test_combine_weights_switch_and_renormalised():
    p = np.array([[0.1, 0.6, 0.3]])
    idx = np.array([[1, 2]], dtype=np.int32)
    assert np.allclose(moe.combine_weights(p, idx), [[0.6, 0.3]])
    assert np.allclose(moe.combine_weights(p, idx, True), [[2 / 3, 1 / 3]])


# ---------------------------------------------------------------- capacity (R4) -------

def test_capacity_formula_cases():
    assert moe.capacity(16384, 2, 8, 1.25) == 5120         # SURVEY cfg2
    assert moe.capacity(32, 2, 4, 1.25) == 20              # tiny
    assert moe.capacity(64, 2, 4, 1.25) == 40
    assert moe.capacity(10, 1, 3, 1.0) == 4                # ceil(10/3)
    assert moe.capacity(5, 2, 2, 100.0) == 5               # clamped to T
    assert moe.capacity(1, 1, 64, 0.01) == 1               # at least 1


# ---------------------------------------------------------------- slotting (R7/R8) ----

def _slots_per_expert(idx, E, C):
    """Independent formulation: for each expert, list its pairs in (t, j) order; admit the
    first C."""
    slot = np.full(idx.shape, -1, dtype=np.int32)
    for e in range(E):
        pairs = [(t, j) for t in range(idx.shape[0]) for j in range(idx.shape[1]) if idx[t, j] == e]
        for s, (t, j) in enumerate(pairs[:C]):
            slot[t, j] = s
    return slot


def _random_idx(T, E, k, skew=1.0):
    l = rng.standard_normal((T, E)) + np.linspace(0, skew * 2, E)[None, :]
    return moe.topk(l.astype(np.float32), k)


@pytest.mark.parametrize("T,E,k,C", [(50, 4, 1, 7), (64, 4, 2, 20), (100, 8, 2, 9), (33, 3, 3, 5)])
def test_slots_match_per_expert_formulation(T, E, k, C):
    idx = _random_idx(T, E, k)
    slot, used = moe.assign_slots(idx, E, C)
    assert np.array_equal(slot, _slots_per_expert(idx, E, C))
    assert all(u <= C for u in used)


def test_spec_route_full_examples():
    # E=2, C=2, 3 tokens all argmax expert 0 -> the third is dropped
    idx = np.zeros((3, 1), dtype=np.int32)
    slot, _ = moe.assign_slots(idx, 2, 2)
    assert slot[:, 0].tolist() == [0, 1, -1]
    # C >= B*S -> zero drops for any routing
    idx = _random_idx(40, 4, 2)
    slot, _ = moe.assign_slots(idx, 4, 40)
    assert np.all(slot >= 0)


def test_derived_worked_example(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "derived_worked_example.json")))
    idx = np.array(g["idx"], dtype=np.int32)
    slot, _ = moe.assign_slots(idx, g["E"], g["C"])
    assert slot.tolist() == g["slot"]
    assert moe.chunk_counts(idx, slot, g["E"], g["n_chunks"]).tolist() == g["chunk_counts"]
    s2, c2 = moe.route_micro(idx, g["E"], g["C"], g["n_chunks"])
    assert s2.tolist() == g["slot"] and c2.tolist() == g["chunk_counts"]
    # the reading matters: GShard's choice-major order admits a different set
    assert g["choice_major_slot_GShard_for_contrast"] != g["slot"]


def test_paper_three_quarter_one_quarter_example():
    # one expert, capacity C = 8; micro-batch 1 holds 3/4 C = 6 of its
    # tokens, micro-batch 2 holds 1/4 C = 2.  Unpartitioned: no drop.  Capacity passing: no
    # drop.  Direct micro-batching with C/2 per micro-batch: 1/4 C = 2 dropped (from mb 1).
    C = 8
    idx = np.array([[0]] * 6 + [[1]] * 2 + [[0]] * 2 + [[1]] * 6, dtype=np.int32)  # 8 | 8 tokens
    full, _ = moe.assign_slots(idx, 2, C)
    assert np.count_nonzero((idx == 0) & (full < 0)) == 0
    passed, counts = moe.route_micro(idx, 2, C, 2)
    assert np.array_equal(passed, full)
    assert counts[0].tolist() == [6, 2]
    naive = moe.route_micro_naive(idx, 2, C // 2, 2)
    dropped = (idx == 0) & (naive < 0)
    assert np.count_nonzero(dropped) == C // 4
    assert np.count_nonzero(dropped[:8]) == C // 4           # all from the first micro-batch


def test_capacity_passing_equals_unpartitioned_1000_trials():
    # SPEC.md L558 / L581: route_micro == route_full for every split, over seeded trials
    r = np.random.default_rng(7)
    for trial in range(1000):
        T = int(r.integers(1, 48))
        E = int(r.integers(2, 9))
        k = int(r.integers(1, min(3, E) + 1))
        cf = float(r.choice([0.25, 0.5, 1.0, 1.25, 2.0]))
        n = int(r.integers(1, min(T, 8) + 1))
        l = r.standard_normal((T, E)) + np.linspace(0, 3 * r.random(), E)
        idx = moe.topk(l.astype(np.float32), k)
        C = moe.capacity(T, k, E, cf)
        full, _ = moe.assign_slots(idx, E, C)
        micro, counts = moe.route_micro(idx, E, C, n)
        assert np.array_equal(full, micro), trial
        assert np.array_equal(counts, moe.chunk_counts(idx, full, E, n)), trial


def test_chunk_counts_prefix_identity():
    # n[e][c] = min(C, P_e(t_{c+1})) - min(C, P_e(t_c)), P_e(t) = pairs routed to e before t
    # -- the identity the GPU slot scan uses; checked against the oracle.
    for _ in range(200):
        T, E, k = int(rng.integers(1, 60)), int(rng.integers(2, 9)), 2
        k = min(k, E)
        idx = _random_idx(T, E, k, skew=2.0)
        C = moe.capacity(T, k, E, float(rng.choice([0.5, 1.0, 1.25])))
        n = int(rng.integers(1, min(T, 8) + 1))
        slot, _ = moe.assign_slots(idx, E, C)
        b = moe.chunk_bounds(T, n)
        P = lambda e, t: int(np.count_nonzero(idx[:t] == e))
        want = np.array([[min(C, P(e, b[c + 1])) - min(C, P(e, b[c])) for c in range(n)]
                         for e in range(E)])
        assert np.array_equal(moe.chunk_counts(idx, slot, E, n), want)


def test_chunk_bounds():
    for T in [1, 2, 7, 64, 1000, 16384]:
        for n in range(1, min(T, 8) + 1):
            b = moe.chunk_bounds(T, n)
            sizes = np.diff(b)
            assert b[0] == 0 and b[-1] == T and len(sizes) == n
            assert sizes.max() - sizes.min() <= 1
            assert list(sizes) == sorted(sizes, reverse=True)        # larger first


# ---------------------------------------------------------------- size matrix ---------

def test_size_matrix_all_local_is_diagonal():
    G, E_l, T, n = 4, 2, 20, 2
    E = G * E_l
    sends = []
    for r in range(G):
        idx = (r * E_l + np.arange(T)[:, None] % E_l).astype(np.int32)   # only local experts
        slot, _ = moe.assign_slots(idx, E, moe.capacity(T, 1, E, 100.0))
        sends.append(moe.chunk_counts(idx, slot, E, n))
    N = moe.size_matrix(sends, G)
    for c in range(n):
        assert np.count_nonzero(N[:, :, c] - np.diag(np.diag(N[:, :, c]))) == 0
        assert np.diag(N[:, :, c]).sum() == G * moe.chunk_bounds(T, n)[c + 1] - G * moe.chunk_bounds(T, n)[c]


def test_size_matrix_uniform_and_conservation():
    G, E_l, T = 4, 2, 64
    E = G * E_l
    sends, admitted = [], []
    for r in range(G):
        idx = (np.arange(T)[:, None] % E).astype(np.int32)               # uniform routing
        slot, _ = moe.assign_slots(idx, E, moe.capacity(T, 1, E, 1.0))
        sends.append(moe.chunk_counts(idx, slot, E, 1))
        admitted.append(int(np.count_nonzero(slot >= 0)))
    N = moe.size_matrix(sends, G)[:, :, 0]
    assert np.all(N == T // G)
    # skewed routing with drops: row sums = admitted per source; per (src, expert) <= C
    sends, admitted = [], []
    for r in range(G):
        idx = _random_idx(T, E, 2, skew=3.0)
        C = moe.capacity(T, 2, E, 0.75)
        slot, _ = moe.assign_slots(idx, E, C)
        cnt = moe.chunk_counts(idx, slot, E, 3)
        assert np.all(cnt.sum(1) <= C)
        sends.append(cnt)
        admitted.append(int(np.count_nonzero(slot >= 0)))
    N = moe.size_matrix(sends, G)
    assert N.sum(axis=(1, 2)).tolist() == admitted
    for dst in range(G):
        R = moe.recv_counts(sends, G, dst)
        assert R.sum() == N[:, dst, :].sum()
        assert R.sum() <= G * E_l * C
