"""Pins of the oracle's Random gate (R18): the SplitMix64 reference
outputs, the counter form equal to the sequential generator, distinct uniform draws,
closed-form cases, partition independence, and the backward by central differences (the
routing does not depend on x or Wg, so the loss is smooth and dWg is exactly zero)."""
import numpy as np
import pytest

from oracle import moe

M64 = (1 << 64) - 1


def test_splitmix64_reference_outputs():
    # the first outputs of SplitMix64 seeded with 0 (Steele, Lea, Flood, OOPSLA 2014; the
    # reference splitmix64.c and java.util.SplittableRandom): e220a8397b1dcdaf, 6e789e6aa1b965f4,
    # 06c45d188009454f
    assert [moe.splitmix64(i, 0) for i in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                                         0x06C45D188009454F]


def test_counter_form_equals_sequential_generator():
    for seed in (0, 1, 12345, (1 << 63) + 17):
        x = seed
        for key in range(200):
            x = (x + 0x9E3779B97F4A7C15) & M64          # stateful: advance, then finalise
            z = x
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
            z ^= z >> 31
            assert moe.splitmix64(key, seed) == z


@pytest.mark.parametrize("E,k", [(8, 1), (8, 2), (5, 3), (4, 4), (64, 2)])
def test_draws_are_distinct_and_weights_uniform(E, k):
    idx, w = moe.random_gate(500, E, k, seed=7)
    assert all(len(set(row)) == k for row in idx.tolist())
    assert idx.min() >= 0 and idx.max() < E
    assert np.all(w == 1.0 / k)
    if k == E:                                            # every token: a permutation of the experts
        assert np.all(np.sort(idx, axis=1) == np.arange(E))


def test_single_expert_and_hand_trace():
    idx, _ = moe.random_gate(10, 1, 1, seed=3)
    assert np.all(idx == 0)
    # hand trace: t = 0, E = 4, k = 2, seed = 0: r0 = 0xe220a8397b1dcdaf mod 4 = 3 -> expert 3;
    # r1 = splitmix64(1) = 0x6e789e6aa1b965f4 mod 3 = 0 -> first of [0, 1, 2] = 0
    idx, _ = moe.random_gate(1, 4, 2, seed=0)
    assert 0xE220A8397B1DCDAF % 4 == 3 and 0x6E789E6AA1B965F4 % 3 == 0
    assert idx.tolist() == [[3, 0]]


def test_draws_are_uniform():
    # chi-square over E = 8 bins, 16000 draws: the 99.99th percentile of chi2(7) is 29.9
    T, E = 16000, 8
    for k in (1, 2):
        idx, _ = moe.random_gate(T, E, k, seed=11)
        for j in range(k):
            c = np.bincount(idx[:, j], minlength=E)
            chi2 = float(np.sum((c - T / E) ** 2 / (T / E)))
            assert chi2 < 29.9, (k, j, chi2)


def test_partition_independent_and_token_major_slots():
    r = np.random.default_rng(0)
    x = r.standard_normal((300, 16)).astype(np.float32)
    wg = r.standard_normal((16, 8)).astype(np.float32)
    rt = moe.route_rank(x, wg, 2, 0.75, 4, gate="random", seed=5)
    # the draws of a token do not depend on the batch around it
    idx_part, _ = moe.random_gate(150, 8, 2, seed=5)
    assert np.array_equal(rt.idx[:150], idx_part)
    slot, _ = moe.assign_slots(rt.idx, 8, rt.C)
    assert np.array_equal(rt.slot, slot) and np.any(rt.slot < 0)
    micro, counts = moe.route_micro(rt.idx, 8, rt.C, 4)
    assert np.array_equal(micro, rt.slot) and np.array_equal(counts, rt.counts)
    assert np.all(rt.logits == 0)


def test_random_gate_backward_by_central_differences():
    G, T, d, f, E, k, cf, seed = 1, 10, 5, 7, 4, 2, 0.6, 9
    r = np.random.default_rng(4)
    xs = [r.standard_normal((T, d))]
    wg = r.standard_normal((d, E))
    w1 = [r.standard_normal((E, f, d)) * 0.5]
    w2 = [r.standard_normal((E, d, f)) * 0.5]
    dys = [r.standard_normal((T, d))]

    def loss():
        res = moe.forward(xs, wg, w1, w2, k, cf, 1, gate="random", seed=seed)
        return float(np.sum(dys[0] * res.y[0])), res

    L0, res = loss()
    assert np.any(res.routing[0].slot < 0)
    g = moe.backward(res, xs, wg, w1, w2, dys)
    assert np.all(g["dwg"][0] == 0)
    h = 1e-6
    for arr, ana in ((xs[0], g["dx"][0]), (w1[0], g["dw1"][0]), (w2[0], g["dw2"][0])):
        num = np.zeros_like(arr)
        for i in np.ndindex(arr.shape):
            v = arr[i]
            arr[i] = v + h; lp, _ = loss()
            arr[i] = v - h; lm, _ = loss()
            arr[i] = v
            num[i] = (lp - lm) / (2 * h)
        assert np.max(np.abs(num - ana)) <= 1e-6 * max(1.0, np.max(np.abs(ana)))
