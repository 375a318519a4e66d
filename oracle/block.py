"""Plain CPU oracle of the GPT-MoE block with pre-MoE partitioning (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference) may
import this module.  It shares no code with paper_2404_19429_b200/ (the CUDA path) and never
imports it; inputs come from synthetic/.

What it computes (BASELINE.json configs[3]).  The paper evaluates MoE
versions of GPT-2 from Huggingface transformers, whose block is pre-LN:

    h   = x + Attn(LN1(x))            self-attention before the MoE layer (L172)
    out = h + MoE(LN2(h))             the MoE layer in place of the MLP (L108)

with Attn = fused q|k|v projection ("kqv", L156), causal multi-head softmax attention and the
output projection ("o", L156).  Readings where the paper is silent (R19-R22): no
projection biases (as the experts, R5), LayerNorm eps 1e-5 with fp32 gain and bias, score
scale 1/sqrt(head_dim), and the GPU's bf16 storage points (a1, qkv, att, o, h, u, out) are
mirrored by rounding there (R22), so that the gate input -- and therefore routing -- matches
the GPU's up to accumulation order.

Lancet partitions the non-MoE computation before the MoE layer along the batch dimension and
gates each partition with the capacity left by the earlier ones (L252-L257, fig:part_all;
Switch and Random gates allow it, L271).  That partitioned evaluation is `block_forward_
chunked`; "mathematical equivalence" (L88) and "the exact token-to-expert mapping and token
dropping as the un-partitioned case" (L256) say it equals the plain block (`block_forward`),
which a CPU test checks.

Floating point: fp64 everywhere (numpy matmul as a library primitive), except the MoE gate
logits (oracle.moe, R1) and the bf16 storage rounding above.  Backward by the chain
rule, pinned by central finite differences and by torch autograd (tests/test_oracle_block.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import moe

LN_EPS = 1e-5


def bf16(a: np.ndarray) -> np.ndarray:
    """Round to the nearest bfloat16 (ties to even), returned as float64 (R22 storage points).
    Through float32 first; the double rounding can only matter for values within 2^-24 of a
    bf16 halfway point."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def _keep(a: np.ndarray, storage: str) -> np.ndarray:
    return bf16(a) if storage == "bf16" else np.asarray(a, dtype=np.float64)


# ----------------------------------------------------------------------------------------
# Non-MoE operators
# ----------------------------------------------------------------------------------------

def layer_norm(x: np.ndarray, g: np.ndarray, b: np.ndarray, eps: float = LN_EPS):
    """GPT-2's LayerNorm (R19): xhat = (x - mean) / sqrt(var + eps) over the last axis
    (biased variance), y = xhat * g + b.  Returns (y, mean, rstd)."""
    x = x.astype(np.float64)
    mu = x.mean(axis=1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    return (x - mu) * rstd * g.astype(np.float64) + b.astype(np.float64), mu[:, 0], rstd[:, 0]


def layer_norm_backward(dy: np.ndarray, x: np.ndarray, g: np.ndarray, mu: np.ndarray, rstd: np.ndarray):
    """Chain rule of layer_norm: dxhat = dy g; dx = rstd (dxhat - mean(dxhat) -
    xhat mean(dxhat xhat)); dg = sum_t dy xhat; db = sum_t dy."""
    xhat = (x.astype(np.float64) - mu[:, None]) * rstd[:, None]
    dxhat = dy * g.astype(np.float64)
    dx = rstd[:, None] * (dxhat - dxhat.mean(axis=1, keepdims=True)
                          - xhat * (dxhat * xhat).mean(axis=1, keepdims=True))
    return dx, (dy * xhat).sum(axis=0), dy.sum(axis=0)


def split_qkv(qkv: np.ndarray, n_heads: int):
    """[T, 3d] (q | k | v; head h at columns h*hd .. h*hd+hd-1 of each) -> q, k, v as
    [T, H, hd]."""
    T, d3 = qkv.shape
    d = d3 // 3
    hd = d // n_heads
    return (qkv[:, :d].reshape(T, n_heads, hd), qkv[:, d:2 * d].reshape(T, n_heads, hd),
            qkv[:, 2 * d:].reshape(T, n_heads, hd))


def causal_attention(qkv: np.ndarray, n_heads: int, seq_len: int):
    """Causal multi-head softmax attention per sequence (GPT-2 self-attention, L172, R19):
    s_ij = <q_i, k_j> / sqrt(hd) for j <= i, p_i = softmax_j(s_i), o_i = sum_j p_ij v_j.
    qkv [T, 3d] with T a multiple of seq_len (sequences are consecutive).  Returns
    (o [T, d], lse [H, T]) with lse the natural-log row normaliser log sum_j exp(s_ij)."""
    T = qkv.shape[0]
    q, k, v = split_qkv(qkv.astype(np.float64), n_heads)
    hd = q.shape[2]
    o = np.zeros_like(q)
    lse = np.zeros((n_heads, T))
    mask = np.tril(np.ones((seq_len, seq_len), dtype=bool))
    for s0 in range(0, T, seq_len):
        sl = slice(s0, s0 + seq_len)
        for h in range(n_heads):
            s = q[sl, h] @ k[sl, h].T / np.sqrt(hd)
            s = np.where(mask, s, -np.inf)
            m = s.max(axis=1, keepdims=True)
            z = np.exp(s - m)
            l = z.sum(axis=1, keepdims=True)
            o[sl, h] = (z / l) @ v[sl, h]
            lse[h, sl] = (m + np.log(l))[:, 0]
    return o.reshape(T, -1), lse


def causal_attention_backward(datt: np.ndarray, qkv: np.ndarray, n_heads: int, seq_len: int):
    """Chain rule of causal_attention: with P the masked softmax, dv = P^T do,
    dP = do v^T, ds = P (dP - rowsum(dP P)), dq = ds k / sqrt(hd), dk = ds^T q / sqrt(hd).
    Returns dqkv [T, 3d]."""
    T = qkv.shape[0]
    q, k, v = split_qkv(qkv.astype(np.float64), n_heads)
    hd = q.shape[2]
    do = datt.astype(np.float64).reshape(T, n_heads, hd)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    mask = np.tril(np.ones((seq_len, seq_len), dtype=bool))
    for s0 in range(0, T, seq_len):
        sl = slice(s0, s0 + seq_len)
        for h in range(n_heads):
            s = np.where(mask, q[sl, h] @ k[sl, h].T / np.sqrt(hd), -np.inf)
            p = np.exp(s - s.max(axis=1, keepdims=True))
            p /= p.sum(axis=1, keepdims=True)
            dv[sl, h] = p.T @ do[sl, h]
            dp = do[sl, h] @ v[sl, h].T
            ds = p * (dp - (dp * p).sum(axis=1, keepdims=True))
            dq[sl, h] = ds @ k[sl, h] / np.sqrt(hd)
            dk[sl, h] = ds.T @ q[sl, h] / np.sqrt(hd)
    return np.concatenate([dq.reshape(T, -1), dk.reshape(T, -1), dv.reshape(T, -1)], axis=1)


# ----------------------------------------------------------------------------------------
# The block over G simulated ranks
# ----------------------------------------------------------------------------------------

@dataclass
class BlockResult:
    out: list                 # [T, d] per rank
    h: list                   # residual after attention, [T, d] per rank
    u: list                   # MoE input LN2(h) (the gate input), [T, d] per rank
    moe: moe.LayerResult      # the MoE layer on u
    saved: dict = field(default_factory=dict)   # per rank: a1, qkv, att, lse, ln stats


def attention_part(x: np.ndarray, p: dict, n_heads: int, seq_len: int, storage: str = "bf16"):
    """The non-MoE computation before the gate for one rank's tokens (whole sequences):
    a1 = LN1(x); qkv = a1 W_qkv^T; att = Attn(qkv); o = att W_o^T; h = x + o; u = LN2(h)."""
    x = x.astype(np.float64)
    a1, mu1, rs1 = layer_norm(x, p["ln1_g"], p["ln1_b"])
    a1 = _keep(a1, storage)
    qkv = _keep(a1 @ p["w_qkv"].astype(np.float64).T, storage)
    att, lse = causal_attention(qkv, n_heads, seq_len)
    att = _keep(att, storage)
    o = _keep(att @ p["w_o"].astype(np.float64).T, storage)
    h = _keep(x + o, storage)
    u, mu2, rs2 = layer_norm(h, p["ln2_g"], p["ln2_b"])
    u = _keep(u, storage)
    return h, u, dict(a1=a1, qkv=qkv, att=att, lse=lse, mu1=mu1, rs1=rs1, mu2=mu2, rs2=rs2)


def block_forward(xs, params, wg, w1_ranks, w2_ranks, n_heads, seq_len, k, cf, n_chunks,
                  act="gelu_tanh", storage="bf16", token_subset=None, experts=None,
                  gate_fp64=False) -> BlockResult:
    """The plain (unpartitioned) block over G = len(xs) ranks: the non-MoE part on each rank's
    whole batch, then oracle.moe.forward on the MoE inputs u (routing per rank over its whole
    batch; n_chunks only labels the per-chunk counts), out = h + y.  `token_subset` /
    `experts` restrict the MoE expert math as in oracle.moe.forward (out rows of other tokens
    are NaN); `gate_fp64` as there (the smooth gate of the finite-difference pins)."""
    hs, us, saved = [], [], {}
    for r, x in enumerate(xs):
        h, u, sv = attention_part(x, params, n_heads, seq_len, storage)
        hs.append(h)
        us.append(u)
        saved[r] = sv
    res = moe.forward(us, wg, w1_ranks, w2_ranks, k, cf, n_chunks, act=act, token_subset=token_subset,
                      experts=experts, gate_fp64=gate_fp64)
    outs = [_keep(h + y, storage) for h, y in zip(hs, res.y)]
    return BlockResult(out=outs, h=hs, u=us, moe=res, saved=saved)


def seq_chunk_bounds(n_seq: int, seq_len: int, n_chunks: int) -> list[int]:
    """Token boundaries of the pre-MoE partition (R20): n_chunks contiguous groups of whole
    sequences (self-attention mixes the tokens of a sequence, so a partition along the batch
    dimension, L252, cuts between sequences), n_seq / n_chunks sequences each."""
    if n_seq % n_chunks:
        raise ValueError("n_chunks must divide the sequences per rank")
    per = n_seq // n_chunks
    return [c * per * seq_len for c in range(n_chunks + 1)]


def block_forward_chunked(xs, params, wg, w1_ranks, w2_ranks, n_heads, seq_len, k, cf, n_chunks,
                          act="gelu_tanh", storage="bf16"):
    """Lancet's partitioned forward (fig:part_all, L252-L257), step by step: for chunk c of
    every rank, the non-MoE part on the chunk's sequences only, the gate on the chunk's tokens
    (logits, top-k, weights per token), admission with the capacity state carried over from
    chunks 0..c-1 ("when the first partition uses 3/4 C, the second will adjust its remaining
    capacity to 1/4 C", L255; oracle.moe.assign_slots with `used`), the chunk's experts and the
    combine.  C comes from the rank's whole batch (R4).  Returns (out per rank, idx per rank,
    slot per rank, per-chunk counts [E][n] per rank)."""
    G = len(xs)
    E = wg.shape[1]
    E_l = E // G
    outs, idxs, slots, counts = [], [], [], []
    for r, x in enumerate(xs):
        T = x.shape[0]
        C = moe.capacity(T, k, E, cf)
        b = seq_chunk_bounds(T // seq_len, seq_len, n_chunks)
        used = [0] * E
        out = np.zeros((T, x.shape[1]))
        idx_r = np.zeros((T, k), np.int32)
        slot_r = np.zeros((T, k), np.int32)
        cnt = np.zeros((E, n_chunks), np.int64)
        for c in range(n_chunks):
            sl = slice(b[c], b[c + 1])
            h, u, _ = attention_part(x[sl], params, n_heads, seq_len, storage)
            logits = moe.gate_logits(u.astype(np.float32), wg)
            idx = moe.topk(logits, k)
            w = moe.combine_weights(moe.softmax(logits), idx)
            before = list(used)
            slot, used = moe.assign_slots(idx, E, C, used)
            for e in range(E):
                cnt[e, c] = used[e] - before[e]
            y = np.zeros_like(h)
            for e in range(E):
                t_sel, j_sel = np.nonzero((idx == e) & (slot >= 0))
                if t_sel.size == 0:
                    continue
                w1e, w2e = moe.expert_weights(w1_ranks, w2_ranks, e, E_l)
                if act == "identity_expert":
                    o = u[t_sel]
                else:
                    _, _, o = moe.expert_ffn(u[t_sel], w1e, w2e, act)
                np.add.at(y, t_sel, w[t_sel, j_sel][:, None] * o)
            out[sl] = _keep(h + y, storage)
            idx_r[sl] = idx
            slot_r[sl] = slot
        outs.append(out)
        idxs.append(idx_r)
        slots.append(slot_r)
        counts.append(cnt)
    return outs, idxs, slots, counts


def block_backward(fwd: BlockResult, xs, params, wg, w1_ranks, w2_ranks, douts, n_heads, seq_len,
                   act="gelu_tanh"):
    """Gradients of sum_r <dout_r, out_r> by the chain rule (no storage rounding):
      dh   = dout + LN2'(du),  du = the MoE layer's input gradient (oracle.moe.backward:
             expert path + gate term)
      dW_o = dh^T att;  datt = dh W_o;  dqkv = Attn'(datt)
      dW_qkv = dqkv^T a1;  da1 = dqkv W_qkv;  dx = dh + LN1'(da1)
    Returns dict(dx, dln1_g, dln1_b, dw_qkv, dw_o, dln2_g, dln2_b [per rank], and the MoE
    layer's dwg, dw1, dw2)."""
    mb = moe.backward(fwd.moe, fwd.u, wg, w1_ranks, w2_ranks, douts, act=act)
    out = {key: [] for key in ("dx", "dln1_g", "dln1_b", "dw_qkv", "dw_o", "dln2_g", "dln2_b")}
    for r, x in enumerate(xs):
        sv = fwd.saved[r]
        dout = douts[r].astype(np.float64)
        du = mb["dx"][r]
        dh2, dg2, db2 = layer_norm_backward(du, fwd.h[r], params["ln2_g"], sv["mu2"], sv["rs2"])
        dh = dout + dh2
        dw_o = dh.T @ sv["att"]
        datt = dh @ params["w_o"].astype(np.float64)
        dqkv = causal_attention_backward(datt, sv["qkv"], n_heads, seq_len)
        dw_qkv = dqkv.T @ sv["a1"]
        da1 = dqkv @ params["w_qkv"].astype(np.float64)
        dx1, dg1, db1 = layer_norm_backward(da1, x, params["ln1_g"], sv["mu1"], sv["rs1"])
        for key, v in (("dx", dh + dx1), ("dln1_g", dg1), ("dln1_b", db1), ("dw_qkv", dw_qkv),
                       ("dw_o", dw_o), ("dln2_g", dg2), ("dln2_b", db2)):
            out[key].append(v)
    out.update(dwg=mb["dwg"], dw1=mb.get("dw1"), dw2=mb.get("dw2"))
    return out
