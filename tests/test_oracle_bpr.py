"""Pins of the oracle's Batch Prioritized Routing (R16) against
things other than itself: closed forms of the importance score, an independent per-expert
formulation, reductions to token-major routing, the paper's "lower scores dropped first"
statement as an invariant, and hand-derived examples."""
import numpy as np
import pytest
import scipy.special

from oracle import moe

rng = np.random.default_rng(4242)


def _logits(T, E, skew=1.0, r=rng):
    return (r.standard_normal((T, E)) + np.linspace(0, 2 * skew, E)[None, :]).astype(np.float32)


# ------------------------------------------------------------ importance score (R16) ----

def test_importance_score_is_sum_of_topk_softmax():
    l = _logits(200, 8)
    for k in (1, 2, 3):
        idx = moe.topk(l, k)
        p = scipy.special.softmax(l.astype(np.float64), axis=1)
        want = np.take_along_axis(p, idx.astype(np.int64), axis=1).sum(axis=1)
        np.testing.assert_allclose(moe.importance_scores(l, idx), want, rtol=1e-14, atol=0)


def test_importance_score_closed_forms():
    # E = 2, k = 1: s = sigmoid(|l0 - l1|)
    l = _logits(100, 2)
    s = moe.importance_scores(l, moe.topk(l, 1))
    np.testing.assert_allclose(s, scipy.special.expit(np.abs(l[:, 0].astype(np.float64) - l[:, 1])),
                               rtol=1e-14)
    # uniform logits: s = k / E exactly representable cases
    l = np.zeros((5, 8), dtype=np.float32)
    for k in (1, 2, 4, 8):
        assert np.all(moe.importance_scores(l, moe.topk(l, k)) == k / 8)
    # k = E: every probability is selected, s = 1 (up to the two summation orders)
    l = _logits(50, 6)
    np.testing.assert_allclose(moe.importance_scores(l, moe.topk(l, 6)), 1.0, rtol=1e-15)


# --------------------------------------------------------------- BPR admission (R16) ----

def _bpr_per_expert(idx, s, E, C):
    """Independent formulation: for each expert, sort ITS pairs by (score desc, t asc) and
    admit the first C; slots = rank of the admitted pairs in token order."""
    slot = np.full(idx.shape, -1, dtype=np.int32)
    for e in range(E):
        pairs = [(t, j) for t in range(idx.shape[0]) for j in range(idx.shape[1]) if idx[t, j] == e]
        adm = sorted(sorted(pairs, key=lambda p: (-s[p[0]], p[0]))[:C])
        for q, (t, j) in enumerate(adm):
            slot[t, j] = q
    return slot


@pytest.mark.parametrize("T,E,k,cf", [(60, 4, 1, 1.0), (64, 4, 2, 0.75), (101, 8, 2, 1.25), (37, 3, 3, 0.5),
                                      (80, 16, 2, 1.0)])
def test_bpr_matches_per_expert_formulation(T, E, k, cf):
    for trial in range(5):
        l = _logits(T, E, skew=1.5)
        idx = moe.topk(l, k)
        s = moe.importance_scores(l, idx)
        C = moe.capacity(T, k, E, cf)
        got = moe.assign_slots_bpr(idx, s, E, C)
        assert np.array_equal(got, _bpr_per_expert(idx, s, E, C)), trial


def test_bpr_lower_scores_dropped_first():
    # "tokens with lower scores would be dropped first"
    for trial in range(30):
        T, E, k = int(rng.integers(20, 120)), int(rng.integers(2, 9)), 2
        l = _logits(T, E, skew=2.0)
        idx = moe.topk(l, k)
        s = moe.importance_scores(l, idx)
        C = moe.capacity(T, k, E, float(rng.choice([0.25, 0.5, 1.0])))
        slot = moe.assign_slots_bpr(idx, s, E, C)
        for e in range(E):
            m = idx == e
            adm, drop = m & (slot >= 0), m & (slot < 0)
            assert np.count_nonzero(adm) == min(C, np.count_nonzero(m))
            if adm.any() and drop.any():
                ts_a, ts_d = np.nonzero(adm)[0], np.nonzero(drop)[0]
                assert s[ts_a].min() >= s[ts_d].max()
            # slots of e are 0..a-1 in token order
            assert np.array_equal(slot[adm], np.arange(np.count_nonzero(adm)))


def test_bpr_equal_scores_reduce_to_token_major():
    # rows are permutations of [0, -1000, ...]: exp(-1000) underflows to 0 in fp64, so every
    # token has s = 1 exactly and BPR's order is the token order (R7 ties by t)
    T, E, k = 90, 5, 2
    l = np.full((T, E), -1000.0, dtype=np.float32)
    l[np.arange(T), rng.integers(0, E, T)] = 0.0
    idx = moe.topk(l, k)
    s = moe.importance_scores(l, idx)
    assert np.all(s == 1.0)
    for C in (3, 10, 40):
        assert np.array_equal(moe.assign_slots_bpr(idx, s, E, C), moe.assign_slots(idx, E, C)[0])


def test_bpr_no_binding_capacity_equals_plain_routing():
    # SPEC.md L548 analogue: C >= T -> no drops; slots are the token-major positions
    l = _logits(70, 4)
    idx = moe.topk(l, 2)
    s = moe.importance_scores(l, idx)
    got = moe.assign_slots_bpr(idx, s, 4, 70)
    assert np.all(got >= 0)
    assert np.array_equal(got, moe.assign_slots(idx, 4, 70)[0])


def test_bpr_hand_example():
    # E = 2, k = 1, C = 2.  Scores and choices (hand-set):
    #   t0: e0 s=.50   t1: e0 s=.90   t2: e1 s=.60   t3: e0 s=.70   t4: e0 s=.90   t5: e1 s=.55
    # e0's pairs by (s desc, t asc): t1(.90) t4(.90) t3(.70) t0(.50) -> admit t1, t4; drop t3, t0
    # e1's pairs: t2, t5 -> both admitted.  Slots in token order: e0: t1->0, t4->1; e1: t2->0, t5->1
    idx = np.array([[0], [0], [1], [0], [0], [1]], dtype=np.int32)
    s = np.array([.50, .90, .60, .70, .90, .55])
    slot = moe.assign_slots_bpr(idx, s, 2, 2)
    assert slot[:, 0].tolist() == [-1, 0, 0, -1, 1, 1]
    # token-major (Switch) routing would instead drop t3 and t4 (the last two of e0)
    assert moe.assign_slots(idx, 2, 2)[0][:, 0].tolist() == [0, 1, 0, -1, -1, 1]


def test_bpr_partition_before_gate_changes_drops():
    # "Splitting along batch dimension would thus cause differences in token
    # dropping".  One expert, C = 2, scores [.1 .2 | .9 .8] in two micro-batches: whole-batch
    # BPR admits t2, t3; sorting each micro-batch separately (capacity passed on) admits t1, t0.
    idx = np.zeros((4, 1), dtype=np.int32)
    s = np.array([.1, .2, .9, .8])
    whole = moe.assign_slots_bpr(idx, s, 1, 2) >= 0
    micro = moe.route_micro_bpr(idx, s, 1, 2, 2)
    assert whole[:, 0].tolist() == [False, False, True, True]
    assert micro[:, 0].tolist() == [True, True, False, False]


def test_bpr_partition_after_gate_chunks_are_contiguous_slot_ranges():
    # partition after the gate (fig:part_after_gate): chunk c's admitted rows of expert e are
    # slots [S_c, S_c+1) with S_c = admitted pairs of e before the chunk -- the same prefix
    # identity the Switch path's capacity passing uses
    for trial in range(100):
        T, E = int(rng.integers(8, 80)), int(rng.integers(2, 7))
        k = min(2, E)
        l = _logits(T, E, skew=2.0)
        idx = moe.topk(l, k)
        s = moe.importance_scores(l, idx)
        C = moe.capacity(T, k, E, 0.5)
        slot = moe.assign_slots_bpr(idx, s, E, C)
        n = int(rng.integers(1, min(T, 8) + 1))
        b = moe.chunk_bounds(T, n)
        counts = moe.chunk_counts(idx, slot, E, n)
        for e in range(E):
            for c in range(n):
                sl = slot[b[c]:b[c + 1]][idx[b[c]:b[c + 1]] == e]
                sl = np.sort(sl[sl >= 0])
                start = int(counts[e, :c].sum())
                assert np.array_equal(sl, np.arange(start, start + counts[e, c]))


def test_route_rank_bpr_and_switch_agree_without_drops():
    l_rank = moe.route_rank(rng.standard_normal((40, 8)).astype(np.float32),
                            rng.standard_normal((8, 4)).astype(np.float32), 2, 4.0, 2, gate="bpr")
    s_rank = moe.route_rank(rng.standard_normal((40, 8)).astype(np.float32),
                            rng.standard_normal((8, 4)).astype(np.float32), 2, 4.0, 2)
    assert np.all(l_rank.slot >= 0) and np.all(s_rank.slot >= 0)
    with pytest.raises(ValueError):
        moe.route_rank(np.zeros((4, 8), np.float32), np.zeros((8, 4), np.float32), 1, 1.0, 1, gate="x")
