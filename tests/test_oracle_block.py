"""Pins of the GPT-MoE block oracle (oracle/block.py) against things other than itself:
torch's LayerNorm, scaled-dot-product attention and autograd (library cross-checks in fp64),
closed forms of causal attention, causality, the dense-mixture special case of the MoE part,
central finite differences, and Lancet's pre-MoE partition equivalence."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synthetic as S
from oracle import block as B
from oracle import moe as M


def _rng(seed):
    return np.random.default_rng(seed)


def test_layer_norm_matches_torch_and_normalises():
    r = _rng(1)
    x = r.standard_normal((37, 96)) * 3 + 1.5
    g, b = 1 + 0.1 * r.standard_normal(96), 0.1 * r.standard_normal(96)
    y, mu, rs = B.layer_norm(x, g, b)
    ref = F.layer_norm(torch.from_numpy(x), (96,), torch.from_numpy(g), torch.from_numpy(b), eps=1e-5)
    assert np.allclose(y, ref.numpy(), rtol=0, atol=1e-12)
    y0, _, _ = B.layer_norm(x, np.ones(96), np.zeros(96))
    assert np.allclose(y0.mean(axis=1), 0, atol=1e-12)
    assert np.allclose((y0 ** 2).mean(axis=1) * (1 + 1e-5 * rs ** 2), 1, atol=1e-9)   # var/(var+eps)


def test_layer_norm_backward_matches_autograd():
    r = _rng(2)
    x = r.standard_normal((9, 40))
    g, b, dy = 1 + 0.1 * r.standard_normal(40), 0.1 * r.standard_normal(40), r.standard_normal((9, 40))
    _, mu, rs = B.layer_norm(x, g, b)
    dx, dg, db = B.layer_norm_backward(dy, x, g, mu, rs)
    xt, gt, bt = (torch.from_numpy(a).requires_grad_() for a in (x, g, b))
    (F.layer_norm(xt, (40,), gt, bt, eps=1e-5) * torch.from_numpy(dy)).sum().backward()
    for mine, ref in ((dx, xt.grad), (dg, gt.grad), (db, bt.grad)):
        assert np.allclose(mine, ref.numpy(), rtol=0, atol=1e-11)


def _sdpa(qkv, H, S_):
    """torch reference: per sequence, [H, S, hd] causal SDPA (fp64)."""
    T = qkv.shape[0]
    q, k, v = (torch.from_numpy(a) for a in B.split_qkv(qkv, H))
    outs = []
    for s0 in range(0, T, S_):
        sl = slice(s0, s0 + S_)
        o = F.scaled_dot_product_attention(q[sl].transpose(0, 1), k[sl].transpose(0, 1), v[sl].transpose(0, 1),
                                           is_causal=True)
        outs.append(o.transpose(0, 1).reshape(S_, -1))
    return torch.cat(outs).numpy()


def test_causal_attention_matches_torch_sdpa():
    r = _rng(3)
    H, S_, hd = 3, 17, 8
    qkv = r.standard_normal((2 * S_, 3 * H * hd))
    o, lse = B.causal_attention(qkv, H, S_)
    assert np.allclose(o, _sdpa(qkv, H, S_), rtol=0, atol=1e-12)
    # lse against torch's logsumexp of the masked scores
    q, k, _ = B.split_qkv(qkv, H)
    s = torch.from_numpy(q[:S_, 1] @ k[:S_, 1].T / np.sqrt(hd))
    s = s.masked_fill(~torch.tril(torch.ones(S_, S_, dtype=torch.bool)), float("-inf"))
    assert np.allclose(lse[1, :S_], torch.logsumexp(s, dim=1).numpy(), atol=1e-12)


def test_causal_attention_closed_forms_and_causality():
    r = _rng(4)
    H, S_, hd = 2, 12, 4
    qkv = r.standard_normal((S_, 3 * H * hd))
    d = H * hd
    o, _ = B.causal_attention(qkv, H, S_)
    # the first token attends only to itself: o_0 = v_0
    assert np.allclose(o[0], qkv[0, 2 * d:], atol=1e-15)
    # q = 0: uniform weights over the prefix, o_i = mean(v_0 .. v_i)
    z = qkv.copy()
    z[:, :d] = 0
    o0, lse0 = B.causal_attention(z, H, S_)
    run = np.cumsum(z[:, 2 * d:], axis=0) / np.arange(1, S_ + 1)[:, None]
    assert np.allclose(o0, run, atol=1e-14)
    assert np.allclose(lse0[0], np.log(np.arange(1, S_ + 1)), atol=1e-14)
    # causality: perturbing token j changes outputs i >= j only
    j = 5
    p = qkv.copy()
    p[j] += 1.0
    op, _ = B.causal_attention(p, H, S_)
    assert np.array_equal(op[:j], o[:j]) and not np.allclose(op[j:], o[j:])
    # sequences do not mix
    two = np.concatenate([qkv, r.standard_normal((S_, 3 * d))])
    o2, _ = B.causal_attention(two, H, S_)
    assert np.allclose(o2[:S_], o, atol=1e-15)


def test_causal_attention_backward_matches_autograd():
    r = _rng(5)
    H, S_, hd = 2, 9, 4
    qkv = r.standard_normal((2 * S_, 3 * H * hd))
    datt = r.standard_normal((2 * S_, H * hd))
    mine = B.causal_attention_backward(datt, qkv, H, S_)
    t = torch.from_numpy(qkv).requires_grad_()
    q, k, v = t[:, :H * hd], t[:, H * hd:2 * H * hd], t[:, 2 * H * hd:]
    outs = []
    for s0 in range(0, 2 * S_, S_):
        sl = slice(s0, s0 + S_)
        f = lambda a: a[sl].reshape(S_, H, hd).transpose(0, 1)  # noqa: E731
        outs.append(F.scaled_dot_product_attention(f(q), f(k), f(v), is_causal=True).transpose(0, 1).reshape(S_, -1))
    (torch.cat(outs) * torch.from_numpy(datt)).sum().backward()
    assert np.allclose(mine, t.grad.numpy(), rtol=0, atol=1e-12)


def _tiny(beta=0.5, **kw):
    sh = S.BlockShape(**{**S.TINY_BLOCK.__dict__, **kw})
    ins = [S.gen_block_rank_inputs(7, r, sh, beta=beta) for r in range(sh.G)]
    p = {key: ins[0][key] for key in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "w_qkv", "w_o")}
    return sh, ins, p


def _torch_block(x, p, wg, w1, w2, H, S_, act):
    """An independent fp64 GPT-2-style block with a DENSE softmax mixture of all experts
    (the MoE layer with k = E and capacity not binding: every choice admitted, R3 weights)."""
    d = x.shape[1]
    T = x.shape[0]
    a1 = F.layer_norm(x, (d,), p["ln1_g"], p["ln1_b"], eps=1e-5)
    qkv = a1 @ p["w_qkv"].T
    q, k, v = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
    hd = d // H
    att = []
    for s0 in range(0, T, S_):
        sl = slice(s0, s0 + S_)
        f = lambda a: a[sl].reshape(S_, H, hd).transpose(0, 1)  # noqa: E731
        att.append(F.scaled_dot_product_attention(f(q), f(k), f(v), is_causal=True).transpose(0, 1).reshape(S_, d))
    h = x + torch.cat(att) @ p["w_o"].T
    u = F.layer_norm(h, (d,), p["ln2_g"], p["ln2_b"], eps=1e-5)
    prob = torch.softmax(u @ wg, dim=1)
    y = torch.zeros_like(u)
    for e in range(wg.shape[1]):
        a = u @ w1[e].T
        hh = F.gelu(a, approximate="tanh") if act == "gelu_tanh" else torch.relu(a)
        y = y + prob[:, e:e + 1] * (hh @ w2[e].T)
    return h + y


@pytest.mark.parametrize("act", ["gelu_tanh", "relu"])
def test_block_is_gpt2_block_with_dense_mixture(act):
    """k = E, capacity not binding: the oracle block equals an independent torch block
    (LayerNorm, SDPA, dense softmax mixture; fp64 gate in both)."""
    sh, ins, p = _tiny(E=4, k=4, cf=4.0)
    xs = [i["x"] for i in ins]
    w1s, w2s = [i["w1"] for i in ins], [i["w2"] for i in ins]
    res = B.block_forward(xs, p, ins[0]["wg"], w1s, w2s, sh.n_heads, sh.seq_len, sh.k, sh.cf, sh.n_chunks,
                          act=act, storage="fp64", gate_fp64=True)
    w1 = torch.from_numpy(np.concatenate(w1s).astype(np.float64))
    w2 = torch.from_numpy(np.concatenate(w2s).astype(np.float64))
    tp = {key: torch.from_numpy(np.asarray(v, dtype=np.float64)) for key, v in p.items()}
    for r in range(sh.G):
        ref = _torch_block(torch.from_numpy(xs[r].astype(np.float64)), tp,
                           torch.from_numpy(ins[0]["wg"].astype(np.float64)), w1, w2, sh.n_heads, sh.seq_len, act)
        assert np.allclose(res.out[r], ref.numpy(), rtol=0, atol=1e-11)


def test_zero_output_projection_reduces_to_the_moe_layer():
    """W_o = 0: h = x, and the block is x + MoE(LN2(x)) (routing and y of oracle.moe)."""
    sh, ins, p = _tiny()
    p = dict(p, w_o=np.zeros_like(p["w_o"]))
    xs = [i["x"] for i in ins]
    w1s, w2s = [i["w1"] for i in ins], [i["w2"] for i in ins]
    res = B.block_forward(xs, p, ins[0]["wg"], w1s, w2s, sh.n_heads, sh.seq_len, sh.k, sh.cf, sh.n_chunks,
                          storage="fp64")
    us = [B.layer_norm(x.astype(np.float64), p["ln2_g"], p["ln2_b"])[0] for x in xs]
    ref = M.forward(us, ins[0]["wg"], w1s, w2s, sh.k, sh.cf, sh.n_chunks)
    for r in range(sh.G):
        assert np.array_equal(res.moe.routing[r].slot, ref.routing[r].slot)
        assert np.allclose(res.out[r], xs[r] + ref.y[r], rtol=0, atol=1e-13)


@pytest.mark.parametrize("n_chunks", [1, 2, 4])
@pytest.mark.parametrize("cf", [0.5, 1.0])
def test_pre_moe_partition_equals_unpartitioned_block(n_chunks, cf):
    """fig:part_all with capacity passing (L252-L257): the chunked block -- non-MoE part per
    chunk of sequences, gate per chunk, admission with the carried capacity state -- gives the
    unpartitioned block's routing, drops and outputs.  Binding capacity (skewed gate, cf <= 1)
    so drops happen and the carry matters."""
    sh, ins, p = _tiny(beta=1.0, cf=cf, n_chunks=n_chunks)
    xs = [i["x"] for i in ins]
    w1s, w2s = [i["w1"] for i in ins], [i["w2"] for i in ins]
    ref = B.block_forward(xs, p, ins[0]["wg"], w1s, w2s, sh.n_heads, sh.seq_len, sh.k, cf, n_chunks)
    outs, idxs, slots, counts = B.block_forward_chunked(xs, p, ins[0]["wg"], w1s, w2s, sh.n_heads, sh.seq_len,
                                                        sh.k, cf, n_chunks)
    dropped = 0
    for r in range(sh.G):
        assert np.array_equal(idxs[r], ref.moe.routing[r].idx)
        assert np.array_equal(slots[r], ref.moe.routing[r].slot)
        assert np.array_equal(counts[r], ref.moe.routing[r].counts)
        assert np.allclose(outs[r], ref.out[r], rtol=0, atol=0)
        dropped += int((slots[r] < 0).sum())
    assert dropped > 0


def test_partition_without_capacity_passing_differs():
    """The paper's counter-example (L253): per-chunk capacity C/n instead of the carried state
    drops different tokens -- the carry is what makes the partition exact."""
    sh, ins, p = _tiny(beta=1.0, cf=1.0, n_chunks=2)
    x = ins[0]["x"]
    h, u, _ = B.attention_part(x, p, sh.n_heads, sh.seq_len)
    idx = M.topk(M.gate_logits(u.astype(np.float32), ins[0]["wg"]), sh.k)
    C = M.capacity(sh.T, sh.k, sh.E, 1.0)
    passing, _ = M.route_micro(idx, sh.E, C, 2)
    naive = M.route_micro_naive(idx, sh.E, C // 2, 2)
    assert np.array_equal(passing, M.assign_slots(idx, sh.E, C)[0])
    assert not np.array_equal(passing >= 0, naive >= 0)


def _loss(xs, p, wg, w1s, w2s, sh, dys):
    res = B.block_forward(xs, p, wg, w1s, w2s, sh.n_heads, sh.seq_len, sh.k, sh.cf, sh.n_chunks,
                          storage="fp64", gate_fp64=True)
    return sum(float(np.sum(o * dy)) for o, dy in zip(res.out, dys)), res


def test_block_backward_finite_differences():
    """Central differences (h = 1e-6, fp64 gate, routing held by margins) of <dout, out> for
    x, both LayerNorms, W_qkv, W_o, Wg and the expert weights."""
    sh = S.BlockShape(n_seq=2, seq_len=6, d=16, n_heads=2, f=12, E=4, G=1, k=2, cf=4.0, n_chunks=1)
    r = _rng(9)
    xs = [r.standard_normal((sh.T, sh.d))]
    p = dict(ln1_g=1 + 0.1 * r.standard_normal(sh.d), ln1_b=0.1 * r.standard_normal(sh.d),
             ln2_g=1 + 0.1 * r.standard_normal(sh.d), ln2_b=0.1 * r.standard_normal(sh.d),
             w_qkv=0.3 * r.standard_normal((3 * sh.d, sh.d)), w_o=0.3 * r.standard_normal((sh.d, sh.d)))
    wg = 0.5 * r.standard_normal((sh.d, sh.E))
    w1s = [0.3 * r.standard_normal((sh.E, sh.f, sh.d))]
    w2s = [0.3 * r.standard_normal((sh.E, sh.d, sh.f))]
    dys = [r.standard_normal((sh.T, sh.d))]
    _, res = _loss(xs, p, wg, w1s, w2s, sh, dys)
    g = B.block_backward(res, xs, p, wg, w1s, w2s, dys, sh.n_heads, sh.seq_len)
    eps = 1e-6

    def fd(arr, i):
        old = arr.flat[i]
        arr.flat[i] = old + eps
        lp, _ = _loss(xs, p, wg, w1s, w2s, sh, dys)
        arr.flat[i] = old - eps
        lm, _ = _loss(xs, p, wg, w1s, w2s, sh, dys)
        arr.flat[i] = old
        return (lp - lm) / (2 * eps)

    checks = [(xs[0], g["dx"][0]), (p["ln1_g"], g["dln1_g"][0]), (p["ln1_b"], g["dln1_b"][0]),
              (p["w_qkv"], g["dw_qkv"][0]), (p["w_o"], g["dw_o"][0]), (p["ln2_g"], g["dln2_g"][0]),
              (p["ln2_b"], g["dln2_b"][0]), (wg, g["dwg"][0]), (w1s[0], g["dw1"][0]), (w2s[0], g["dw2"][0])]
    for arr, grad in checks:
        idx = r.choice(arr.size, size=min(6, arr.size), replace=False)
        for i in idx:
            num = fd(arr, int(i))
            assert abs(num - grad.flat[int(i)]) <= 1e-6 * max(1.0, abs(num)), (num, grad.flat[int(i)])
