"""Pins of the oracle's layer forward/backward against textbook special cases (dense MLP via
torch.nn.functional), identity experts, invariances and central finite differences."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synthetic as S
from oracle import moe

rng = np.random.default_rng(99)


def _inputs(G, T, d, f, E, beta=0.5, seed=0, dtype="bf16"):
    sh = S.LayerShape(T=T, d=d, f=f, E=E, G=G, k=2, cf=1.25, n_chunks=2)
    ins = [S.gen_rank_inputs(seed, r, sh, beta=beta, dtype=dtype) for r in range(G)]
    return ([i["x"] for i in ins], ins[0]["wg"], [i["w1"] for i in ins], [i["w2"] for i in ins],
            [i["dy"] for i in ins])


def test_identity_experts_reproduce_gate_weighted_inputs():
    # north_star: dispatch followed by combine with identity experts reproduces
    # y_t = (sum over admitted j of w_tj) * x_t; dropped tokens -> 0
    xs, wg, w1, w2, _ = _inputs(2, 64, 16, 32, 4, beta=2.0)
    res = moe.forward(xs, wg, w1, w2, 2, 0.5, 2, act="identity_expert")
    n_dropped = 0
    for r in range(2):
        rt = res.routing[r]
        scale = np.where(rt.slot >= 0, rt.w, 0.0).sum(1)
        assert np.allclose(res.y[r], scale[:, None] * xs[r].astype(np.float64), rtol=1e-15, atol=0)
        n_dropped += int(np.count_nonzero(rt.slot < 0))
    assert n_dropped > 0                                  # the case exercises drops


@pytest.mark.parametrize("act,torch_act", [("gelu_tanh", lambda a: F.gelu(a, approximate="tanh")),
                                           ("relu", F.relu)])
def test_single_expert_is_dense_mlp(act, torch_act):
    # E=1, k=1, cf=1 -> C=T, p=1: the MoE layer is the dense MLP y = act(x W1^T) W2^T
    xs, wg, w1, w2, _ = _inputs(1, 40, 12, 24, 1)
    res = moe.forward(xs, wg, w1, w2, 1, 1.0, 1, act=act)
    x = torch.tensor(xs[0], dtype=torch.float64)
    want = F.linear(torch_act(F.linear(x, torch.tensor(w1[0][0], dtype=torch.float64))),
                    torch.tensor(w2[0][0], dtype=torch.float64))
    assert np.allclose(res.y[0], want.numpy(), rtol=1e-12, atol=1e-15)


def test_non_binding_capacity_is_dense_mixture():
    # cf >= E/k -> nothing dropped -> y_t = sum_j w_tj FFN_{idx_tj}(x_t) for every token,
    # computed per token with torch (no dispatch, no buffers)
    G, T, d, f, E = 2, 24, 8, 16, 4
    xs, wg, w1, w2, _ = _inputs(G, T, d, f, E, beta=1.0)
    res = moe.forward(xs, wg, w1, w2, 2, E / 2, 1)
    Wg = torch.tensor(wg, dtype=torch.float64)
    for r in range(G):
        x = torch.tensor(xs[r], dtype=torch.float64)
        p = torch.softmax(x @ Wg, dim=1)
        idx = res.routing[r].idx
        for t in range(T):
            acc = torch.zeros(d, dtype=torch.float64)
            for j in range(2):
                e = int(idx[t, j])
                W1 = torch.tensor(w1[e // 2][e % 2], dtype=torch.float64)
                W2 = torch.tensor(w2[e // 2][e % 2], dtype=torch.float64)
                acc += p[t, e] * (F.gelu(x[t] @ W1.T, approximate="tanh") @ W2.T)
            # softmax of fp32-chain logits vs fp64 logits: relative difference ~1e-7
            assert np.allclose(res.y[r][t], acc.numpy(), rtol=1e-5, atol=1e-9)


def test_placement_invariance_across_rank_counts():
    # the same global experts placed on 1, 2 or 4 ranks give rank 0 the same output
    T, d, f, E = 32, 8, 16, 4
    x0 = S.gen_tokens(5, 0, T, d)
    wg = S.gen_gate(5, d, E, 0.5)
    W1, W2 = S.gen_experts(5, E, d, f)
    ys = []
    for G in (1, 2, 4):
        E_l = E // G
        xs = [x0] + [S.gen_tokens(5, r, T, d) for r in range(1, G)]
        w1 = [W1[r * E_l:(r + 1) * E_l] for r in range(G)]
        w2 = [W2[r * E_l:(r + 1) * E_l] for r in range(G)]
        ys.append(moe.forward(xs, wg, w1, w2, 2, 1.0, 2).y[0])
    assert np.allclose(ys[0], ys[1], rtol=1e-14, atol=0) and np.allclose(ys[0], ys[2], rtol=1e-14, atol=0)


def test_output_linear_in_w2():
    xs, wg, w1, w2, _ = _inputs(2, 32, 8, 16, 4)
    y1 = moe.forward(xs, wg, w1, w2, 2, 1.25, 2).y
    y2 = moe.forward(xs, wg, w1, [3.0 * w for w in w2], 2, 1.25, 2).y
    for a, b in zip(y1, y2):
        assert np.allclose(b, 3.0 * a, rtol=1e-13, atol=1e-18)


def test_token_subset_matches_full():
    xs, wg, w1, w2, _ = _inputs(2, 48, 8, 16, 4)
    full = moe.forward(xs, wg, w1, w2, 2, 1.25, 2)
    sub = [[0, 5, 47], [1, 2, 30]]
    part = moe.forward(xs, wg, w1, w2, 2, 1.25, 2, token_subset=sub)
    for r in range(2):
        assert np.allclose(part.y[r][sub[r]], full.y[r][sub[r]], rtol=1e-12, atol=1e-18)


def test_expert_restriction_partitions_the_layer():
    # experts=[...] (the cost restriction of the full-size GPU tests): the per-expert forwards
    # sum to the full y, and each restricted backward gives exactly the full dW of its experts
    xs, wg, w1, w2, dys = _inputs(2, 64, 8, 16, 4)
    full = moe.forward(xs, wg, w1, w2, 2, 1.25, 2)
    gfull = moe.backward(full, xs, wg, w1, w2, dys)
    ysum = [np.zeros_like(y) for y in full.y]
    for e in range(4):
        part = moe.forward(xs, wg, w1, w2, 2, 1.25, 2, experts=[e])
        gp = moe.backward(part, xs, wg, w1, w2, dys)
        for r in range(2):
            ysum[r] += part.y[r]
        r, el = e // 2, e % 2
        assert np.allclose(gp["dw1"][r][el], gfull["dw1"][r][el], rtol=1e-12, atol=1e-18)
        assert np.allclose(gp["dw2"][r][el], gfull["dw2"][r][el], rtol=1e-12, atol=1e-18)
        other = 1 - el
        assert not np.any(gp["dw1"][r][other]) and not np.any(gp["dw2"][r][other])
    for r in range(2):
        assert np.allclose(ysum[r], full.y[r], rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------- backward by FD -------

def _loss(xs, wg, w1, w2, dys, k, cf, act, renorm, ref_routing=None):
    res = moe.forward(xs, wg, w1, w2, k, cf, 1, act=act, renormalize=renorm, gate_fp64=True)
    if ref_routing is not None:                           # routing must be held fixed
        for a, b in zip(res.routing, ref_routing):
            assert np.array_equal(a.idx, b.idx) and np.array_equal(a.slot, b.slot)
    return sum(float(np.sum(dy.astype(np.float64) * y)) for dy, y in zip(dys, res.y)), res


@pytest.mark.parametrize("act,renorm", [("gelu_tanh", False), ("gelu_tanh", True),
                                        ("relu", False), ("identity_expert", False)])
def test_backward_matches_central_differences(act, renorm):
    G, T, d, f, E, k = 2, 12, 6, 10, 4, 2
    r = np.random.default_rng(3)
    xs = [r.standard_normal((T, d)) for _ in range(G)]
    wg = r.standard_normal((d, E)) * 0.8
    w1 = [r.standard_normal((E // G, f, d)) * 0.5 for _ in range(G)]
    w2 = [r.standard_normal((E // G, d, f)) * 0.5 for _ in range(G)]
    dys = [r.standard_normal((T, d)) for _ in range(G)]
    cf = 0.6                                               # C = 4 < load: forces drops
    L0, res = _loss(xs, wg, w1, w2, dys, k, cf, act, renorm)
    assert sum(int(np.count_nonzero(rt.slot < 0)) for rt in res.routing) > 0
    grads = moe.backward(res, xs, wg, w1, w2, dys, act=act, renormalize=renorm)
    h = 1e-6

    def fd(get, set_):
        base = get().copy()
        out = np.zeros_like(base)
        for i in np.ndindex(base.shape):
            v = base.copy(); v[i] += h; set_(v)
            lp, _ = _loss(xs, wg_c[0], w1, w2, dys, k, cf, act, renorm, res.routing)
            v = base.copy(); v[i] -= h; set_(v)
            lm, _ = _loss(xs, wg_c[0], w1, w2, dys, k, cf, act, renorm, res.routing)
            out[i] = (lp - lm) / (2 * h)
        set_(base)
        return out

    wg_c = [wg]

    def check(num, ana):
        ana = np.asarray(ana)
        assert np.max(np.abs(num - ana)) <= 1e-6 * max(1.0, np.max(np.abs(ana))), (num, ana)

    for rr in range(G):
        def set_x(v, rr=rr): xs[rr] = v
        check(fd(lambda rr=rr: xs[rr], set_x), grads["dx"][rr])
    def set_wg(v): wg_c[0] = v
    check(fd(lambda: wg_c[0], set_wg), sum(grads["dwg"]))          # replicated gate: DP sum
    if act != "identity_expert":
        for rr in range(G):
            def set_w1(v, rr=rr): w1[rr] = v
            def set_w2(v, rr=rr): w2[rr] = v
            check(fd(lambda rr=rr: w1[rr], set_w1), grads["dw1"][rr])
            check(fd(lambda rr=rr: w2[rr], set_w2), grads["dw2"][rr])
