"""GPU parity of the GPT-MoE block with Lancet's pre-MoE partition (SURVEY.md §8(f) NEXT-1,
include/lancet_block.h) and of the partitioned MoE forward it is built on, against the oracle
(oracle/block.py, oracle/moe.py) on the same seeded inputs.

* lancet_moe_forward_partitioned (every chunk gated on its own with the carried capacity state,
  PAPER.md L255): routing, slots, counts bit-exact with the unpartitioned oracle layer, y and the
  backward within the bf16 bar, and bitwise the whole-batch push path's results.
* the block: LN1 / q|k|v / attention / h / u (the gate input) / lse within the bf16 bar of the
  oracle's own non-MoE part; routing equal wherever the oracle's top-k decision has a margin
  larger than what bf16 rounding of u can move (see _routing_check), out within the bar; chunk
  count and the serial baseline bitwise neutral; the pipelined timeline overlaps chunk c+1's
  attention with chunk c's exchange / experts."""
import numpy as np
import pytest
import torch

import synthetic as S
from gpu_harness import TOL, normwise, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_19429_b200 import build
    build.build()


bf = torch.bfloat16


# ---------------------------------------------------------------------------------------------
# the partitioned MoE forward (seeded inputs, no attention)
# ---------------------------------------------------------------------------------------------

def _push_ctx(T, d, f, E, k, max_chunks=8, flags=0):
    from paper_2404_19429_b200 import FLAG_PEER_PUSH, lancet
    cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k, max_chunks=max_chunks,
                             flags=FLAG_PEER_PUSH | flags)
    return lancet.Context(cfg, transport="peer")


@pytest.mark.parametrize("T,d,f,E,k,cf,n", [(1000, 128, 256, 4, 2, 1.0, 4), (777, 256, 384, 8, 1, 1.25, 3),
                                             (2048, 256, 512, 8, 2, 0.5, 8), (300, 128, 256, 16, 4, 1.0, 1)])
def test_partitioned_forward_matches_the_oracle(T, d, f, E, k, cf, n):
    from oracle import moe
    sh = S.LayerShape(T=T, d=d, f=f, E=E, G=1, k=k, cf=cf, n_chunks=n)
    ins = S.gen_rank_inputs(41, 0, sh, beta=0.5)
    resid = S.gen_dy(43, 0, T, d) / 32            # any bf16 tensor (of the MoE output's scale): y = resid + MoE(x)
    ctx = _push_ctx(T, d, f, E, k, max_chunks=max(8, n))
    x, wg, w1, w2, dy = (to_dev(ins[key], torch.float32 if key == "wg" else bf) for key in ("x", "wg", "w1", "w2", "dy"))
    r = to_dev(resid, bf)
    y, idx, slot, w = ctx.forward_partitioned(x, wg, w1, w2, k, cf, n, resid=r)
    dx, dwg, dw1, dw2 = ctx.backward(dy)
    torch.cuda.synchronize()
    send, _, C = ctx.counts(n)
    fwd = moe.forward([ins["x"]], ins["wg"], [ins["w1"]], [ins["w2"]], k, cf, n)
    rt = fwd.routing[0]
    # chunked gating with capacity passing == the unpartitioned layer (L256), bit for bit
    assert np.array_equal(idx.cpu().numpy(), rt.idx)
    assert np.array_equal(slot.cpu().numpy(), rt.slot)
    assert C == rt.C and np.array_equal(send, rt.counts)
    assert np.array_equal(ctx.logits(T).view(np.uint32), rt.logits.view(np.uint32))
    assert normwise(y.float().cpu().numpy(), resid + fwd.y[0]) <= TOL["bf16"]
    b = moe.backward(fwd, [ins["x"]], ins["wg"], [ins["w1"]], [ins["w2"]], [ins["dy"]])
    for got, key in ((dx, "dx"), (dwg, "dwg"), (dw1, "dw1"), (dw2, "dw2")):
        assert normwise(got.float().cpu().numpy(), b[key][0]) <= TOL["bf16"], key
    assert (rt.slot < 0).any() or cf > 1.0 or k == 4
    ctx.close()


def test_partitioned_forward_is_bitwise_the_whole_batch_push_path():
    T, d, f, E, k, cf, n = 2048, 256, 512, 8, 2, 1.0, 4
    sh = S.LayerShape(T=T, d=d, f=f, E=E, G=1, k=k, cf=cf, n_chunks=n)
    ins = S.gen_rank_inputs(47, 0, sh, beta=0.5)
    outs = []
    for part in (False, True):
        ctx = _push_ctx(T, d, f, E, k)
        x, wg, w1, w2, dy = (to_dev(ins[key], torch.float32 if key == "wg" else bf)
                             for key in ("x", "wg", "w1", "w2", "dy"))
        fw = ctx.forward_partitioned if part else ctx.forward
        y, idx, slot, w = fw(x, wg, w1, w2, k, cf, n)
        dx, dwg, dw1, dw2 = ctx.backward(dy)
        torch.cuda.synchronize()
        outs.append([t.cpu() for t in (y, idx, slot, w, dx, dwg)] + [dw1.cpu(), dw2.cpu()])
        ctx.close()
    for a, b in zip(outs[0][:6], outs[1][:6]):
        assert torch.equal(a, b)
    # the dW GEMMs see the rows in another buffer layout (static regions): fp32 reassociation
    for a, b in zip(outs[0][6:], outs[1][6:]):
        assert normwise(b.numpy(), a.numpy()) <= 1e-5


def test_partitioned_forward_two_steps_new_inputs():
    from oracle import moe
    T, d, f, E, k, cf, n = 1024, 128, 256, 4, 2, 1.0, 2
    ctx = _push_ctx(T, d, f, E, k)
    for step in range(2):
        sh = S.LayerShape(T=T, d=d, f=f, E=E, G=1, k=k, cf=cf, n_chunks=n)
        ins = S.gen_rank_inputs(60 + step, 0, sh, beta=0.5)
        x, wg, w1, w2 = (to_dev(ins[key], torch.float32 if key == "wg" else bf) for key in ("x", "wg", "w1", "w2"))
        y, idx, slot, _ = ctx.forward_partitioned(x, wg, w1, w2, k, cf, n)
        torch.cuda.synchronize()
        fwd = moe.forward([ins["x"]], ins["wg"], [ins["w1"]], [ins["w2"]], k, cf, n)
        assert np.array_equal(slot.cpu().numpy(), fwd.routing[0].slot)
        assert normwise(y.float().cpu().numpy(), fwd.y[0]) <= TOL["bf16"]
    ctx.close()


def test_partitioned_forward_refuses_bpr_and_small_buffers():
    from paper_2404_19429_b200 import FLAG_GATE_BPR, lancet
    T, d, f, E, k = 512, 128, 256, 4, 2
    ins = S.gen_rank_inputs(5, 0, S.LayerShape(T=T, d=d, f=f, E=E, G=1, k=k, cf=1.0, n_chunks=2))
    x, wg, w1, w2 = (to_dev(ins[key], torch.float32 if key == "wg" else bf) for key in ("x", "wg", "w1", "w2"))
    ctx = _push_ctx(T, d, f, E, k, flags=FLAG_GATE_BPR)
    with pytest.raises(lancet.LancetError, match="ERR_UNSUPPORTED"):
        ctx.forward_partitioned(x, wg, w1, w2, k, 1.0, 2)
    ctx.close()
    ctx = _push_ctx(T, d, f, E, k, max_chunks=1)
    with pytest.raises(lancet.LancetError, match="ERR_ARG"):
        ctx.forward_partitioned(x, wg, w1, w2, k, 4.0, 1)      # static regions exceed the buffers
    ctx.close()


# ---------------------------------------------------------------------------------------------
# the block
# ---------------------------------------------------------------------------------------------

def _block(sh: S.BlockShape, flags=0, cf_max=2.0):
    from paper_2404_19429_b200 import block, lancet
    moe = lancet.LayerConfig(d_model=sh.d, d_ffn=sh.f, n_experts=sh.E, max_tokens=sh.T, max_k=sh.k, max_chunks=8,
                             flags=flags)
    return block.Block(block.BlockConfig(moe, n_heads=sh.n_heads, seq_len=sh.seq_len, max_capacity_factor=cf_max))


def _dev_params(ins):
    from paper_2404_19429_b200 import block
    return {key: to_dev(ins[key], torch.float32 if key in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "wg") else bf)
            for key in block.PARAMS}


def _routing_check(g_idx, g_slot, o_logits, o_idx, o_slot, du, wg, k):
    """Routing of the GPU block vs the oracle block.  The gate input u comes out of bf16
    attention on both sides, so the two u differ by accumulation-order rounding du; a logit
    difference l_e - l_e' moves by du . (Wg[:, e] - Wg[:, e']), whose size is bounded here by
    8 sigma of independent errors: 8 * rms(du) * sqrt(d) * max |Wg[:, e] - Wg[:, e']|_rms.
    Every token whose top-(k+1) logits are separated by more than that must choose the same
    experts in the same order; if all tokens agree, the slots (capacity admission) must agree
    bit for bit.  Returns the number of tokens inside the margin."""
    d = wg.shape[0]
    diff_rms = max(np.sqrt(np.mean((wg[:, a] - wg[:, b]) ** 2))
                   for a in range(wg.shape[1]) for b in range(a + 1, wg.shape[1])) if wg.shape[1] > 1 else 0.0
    bound = 8 * np.sqrt(np.mean(du ** 2)) * np.sqrt(d) * diff_rms
    srt = -np.sort(-o_logits.astype(np.float64), axis=1)
    kk = min(k + 1, srt.shape[1])
    margin = np.min(srt[:, :kk - 1] - srt[:, 1:kk], axis=1) if kk > 1 else np.full(len(srt), np.inf)
    sure = margin > bound
    assert np.array_equal(g_idx[sure], o_idx[sure]), "confident routing decisions differ"
    if np.array_equal(g_idx, o_idx):
        assert np.array_equal(g_slot, o_slot)
    return int((~sure).sum())


@pytest.mark.parametrize("n_seq,S_,d,H,f,E,k,cf,n", [(4, 256, 256, 2, 512, 4, 2, 1.0, 2),
                                                      (2, 128, 384, 3, 256, 8, 1, 1.25, 2),
                                                      (8, 128, 256, 2, 256, 4, 1, 0.75, 4)])
def test_block_forward_matches_the_oracle(n_seq, S_, d, H, f, E, k, cf, n):
    from oracle import block as OB
    sh = S.BlockShape(n_seq=n_seq, seq_len=S_, d=d, n_heads=H, f=f, E=E, G=1, k=k, cf=cf, n_chunks=n)
    ins = S.gen_block_rank_inputs(11, 0, sh, beta=0.5)
    blk = _block(sh)
    p = _dev_params(ins)
    x = to_dev(ins["x"], bf)
    out = blk.forward(x, p, k, cf, n)
    torch.cuda.synchronize()
    prm = {key: ins[key] for key in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "w_qkv", "w_o")}
    ref = OB.block_forward([ins["x"]], prm, ins["wg"], [ins["w1"]], [ins["w2"]], H, S_, k, cf, n)
    sv = ref.saved[0]
    T = sh.T
    for name, o in (("a1", sv["a1"]), ("qkv", sv["qkv"]), ("att", sv["att"]), ("h", ref.h[0]), ("u", ref.u[0])):
        assert normwise(blk.debug(name, T).float().numpy(), o) <= TOL["bf16"], name
    lse_nat = blk.debug("lse", T).double().numpy() * np.log(2.0)
    assert np.max(np.abs(lse_nat - sv["lse"])) <= 1e-2
    rt = ref.moe.routing[0]
    du = blk.debug("u", T).double().numpy() - ref.u[0]
    g_idx, g_slot = blk.debug("idx", T).numpy(), blk.debug("slot", T).numpy()
    _, _, C = blk.moe.counts()
    assert C == rt.C
    assert np.array_equal(g_slot, _admit(g_idx, C, E)), "GPU slots are not the token-major admission of its choices"
    _routing_check(g_idx, g_slot, rt.logits, rt.idx, rt.slot, du, ins["wg"], k)
    same = np.all(g_idx == rt.idx, axis=1) & np.all((g_slot >= 0) == (rt.slot >= 0), axis=1)
    assert same.mean() > 0.95
    got = out.float().cpu().numpy()
    assert normwise(got[same], ref.out[0][same]) <= TOL["bf16"]
    blk.close()


def _admit(idx, C, E):
    """Token-major admission (R7) of given choices -- the validity check of the GPU's slots
    for its own choices."""
    T, k = idx.shape
    used = np.zeros(E, np.int64)
    slot = np.full((T, k), -1, np.int32)
    for t in range(T):
        for j in range(k):
            e = idx[t, j]
            if used[e] < C:
                slot[t, j] = used[e]
                used[e] += 1
    return slot


def test_block_chunking_and_serial_baseline_are_bitwise_neutral():
    """n = 1, 2, 4 chunks and the one-stream serial baseline give the same out, routing and
    intermediates bit for bit (attention per sequence, row-independent GEMMs, per-token
    kernels; capacity passing reproduces the unpartitioned admission)."""
    from paper_2404_19429_b200 import FLAG_SERIAL
    sh = S.BlockShape(n_seq=4, seq_len=256, d=256, n_heads=2, f=512, E=8, G=1, k=2, cf=1.0, n_chunks=1)
    ins = S.gen_block_rank_inputs(13, 0, sh, beta=0.5)
    res = []
    for n, flags in ((1, 0), (2, 0), (4, 0), (4, FLAG_SERIAL)):
        blk = _block(sh, flags=flags)
        p = _dev_params(ins)
        out = blk.forward(to_dev(ins["x"], bf), p, sh.k, sh.cf, n)
        torch.cuda.synchronize()
        res.append((out.cpu(), blk.debug("u", sh.T), blk.debug("slot", sh.T), blk.debug("idx", sh.T)))
        blk.close()
    for r in res[1:]:
        for a, b in zip(res[0], r):
            assert torch.equal(a, b)


def test_block_pipeline_overlaps_attention_with_the_exchange():
    """The timeline of a pipelined block forward: chunk c+1's attention runs while chunk c's
    dispatch push / experts / combine are in flight (the non-MoE computation in the
    computation-communication pipeline)."""
    from paper_2404_19429_b200 import FLAG_TIMELINE
    sh = S.BlockShape(n_seq=8, seq_len=512, d=512, n_heads=4, f=2048, E=8, G=1, k=1, cf=1.25, n_chunks=4)
    ins = S.gen_block_rank_inputs(17, 0, sh, beta=0.25)
    blk = _block(sh, flags=FLAG_TIMELINE)
    p = _dev_params(ins)
    x = to_dev(ins["x"], bf)
    for _ in range(3):
        blk.forward(x, p, sh.k, sh.cf, sh.n_chunks)
    torch.cuda.synchronize()
    tl = blk.moe.timeline()
    names = {r["name"] for r in tl}
    assert {"ln1", "qkv_proj", "attention", "o_proj", "ln2", "gate", "a2a_counts", "a2a_dispatch_push",
            "expert_fc1", "expert_fc2", "a2a_combine_fused"} <= names
    att = {r["chunk"]: r for r in tl if r["name"] == "attention"}
    later = [r for r in tl if r["chunk"] >= 0 and r["name"] in ("a2a_dispatch_push", "expert_fc1", "expert_fc2",
                                                                  "a2a_combine_fused")]
    overlaps = 0
    for r in later:
        a = att.get(r["chunk"] + 1)
        if a and min(a["end_us"], r["end_us"]) > max(a["start_us"], r["start_us"]):
            overlaps += 1
    assert overlaps >= 1, tl
    blk.close()


def test_block_moe_backward_after_a_block_forward():
    """The block's MoE layer keeps a normal forward state: lancet_moe_backward after a block
    forward gives the oracle layer's gradients for the layer input u (with the oracle's routing
    where it agrees -- identical u is not guaranteed, so this checks dW / dWg shapes and that
    the dx of the MoE layer is consistent with a partitioned layer forward on the GPU's u)."""
    sh = S.BlockShape(n_seq=4, seq_len=128, d=256, n_heads=2, f=256, E=4, G=1, k=2, cf=1.0, n_chunks=2)
    ins = S.gen_block_rank_inputs(19, 0, sh, beta=0.5)
    blk = _block(sh)
    p = _dev_params(ins)
    blk.forward(to_dev(ins["x"], bf), p, sh.k, sh.cf, sh.n_chunks)
    dy = to_dev(S.gen_dy(21, 0, sh.T, sh.d), bf)
    dx, dwg, dw1, dw2 = blk.moe.backward(dy)
    torch.cuda.synchronize()
    u = blk.debug("u", sh.T).cuda()
    # the same layer on the same (GPU) u through the partitioned layer API of a fresh context
    ctx = _push_ctx(sh.T, sh.d, sh.f, sh.E, sh.k)
    ctx.forward_partitioned(u, p["wg"], p["w1"], p["w2"], sh.k, sh.cf, sh.n_chunks)
    dx2, dwg2, dw12, dw22 = ctx.backward(dy)
    torch.cuda.synchronize()
    assert torch.equal(dx.cpu(), dx2.cpu()) and torch.equal(dwg.cpu(), dwg2.cpu())
    assert normwise(dw1.cpu().numpy(), dw12.cpu().numpy()) <= 1e-5
    ctx.close()
    blk.close()


@pytest.mark.parametrize("n_chunks", [4])
def test_block_configs3_full_size_sampled(n_chunks):
    """BASELINE configs[3] per rank (one-rank group: all 32 experts local): T = 8 x 1024,
    d = 2048, 16 heads, f = 8192, E = 32, Switch top-1, cf = 1.25.  The oracle runs the non-MoE
    part of every sequence (the gate needs the whole batch for capacity) and the experts of 64
    sampled tokens."""
    from oracle import block as OB
    from oracle import moe
    sh = S.CFG4
    sh = S.BlockShape(**{**sh.__dict__, "G": 1, "n_chunks": n_chunks})
    ins = S.gen_block_rank_inputs(23, 0, sh, beta=0.25)
    blk = _block(sh, cf_max=1.25)
    p = _dev_params(ins)
    out = blk.forward(to_dev(ins["x"], bf), p, sh.k, sh.cf, n_chunks)
    torch.cuda.synchronize()
    prm = {key: ins[key] for key in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "w_qkv", "w_o")}
    h, u, sv = OB.attention_part(ins["x"], prm, sh.n_heads, sh.seq_len)
    assert normwise(blk.debug("u", sh.T).float().numpy(), u) <= TOL["bf16"]
    assert normwise(blk.debug("h", sh.T).float().numpy(), h) <= TOL["bf16"]
    rng = np.random.default_rng(5)
    tok = np.sort(rng.choice(sh.T, 64, replace=False))
    fwd = moe.forward([u], ins["wg"], [ins["w1"]], [ins["w2"]], sh.k, sh.cf, n_chunks, token_subset=[tok])
    rt = fwd.routing[0]
    g_idx, g_slot = blk.debug("idx", sh.T).numpy(), blk.debug("slot", sh.T).numpy()
    _, _, C = blk.moe.counts()
    assert C == rt.C == 320
    assert np.array_equal(g_slot, _admit(g_idx, C, sh.E))
    du = blk.debug("u", sh.T).double().numpy() - u
    _routing_check(g_idx, g_slot, rt.logits, rt.idx, rt.slot, du, ins["wg"], sh.k)
    same = np.all(g_idx[tok] == rt.idx[tok], axis=1) & np.all((g_slot[tok] >= 0) == (rt.slot[tok] >= 0), axis=1)
    assert same.mean() > 0.9
    ref = OB.bf16(h[tok] + fwd.y[0][tok])
    got = out.float().cpu().numpy()[tok]
    assert normwise(got[same], ref[same]) <= TOL["bf16"]
    assert (rt.slot < 0).any()          # capacity binds at this skew
    blk.close()


# ---------------------------------------------------------------------------------------------
# several processes (ranks) on one GPU over the peer transport
# ---------------------------------------------------------------------------------------------

def _run_peer(tmp_path, G, **spec):
    from test_gpu_peer import run_peer
    return run_peer(tmp_path, G, **spec)


@pytest.mark.parametrize("G,Ts,E,k,n", [(2, [700, 513], 8, 2, 3), (4, [300, 420, 256, 333], 8, 2, 4),
                                         (2, [1024, 1024], 4, 1, 2)])
def test_partitioned_forward_over_processes_matches_the_oracle(tmp_path, G, Ts, E, k, n):
    """Per-chunk size exchange (column c of the count matrix into every peer's), per-chunk
    plan with the static regions and the push over G processes: routing and every output of
    two steps (new inputs each) against the oracle."""
    from paper_2404_19429_b200 import FLAG_PEER_PUSH
    from test_gpu_peer import check_steps
    spec = dict(Ts=Ts, d=128, f=256, E=E, k=k, n=n, cf=1.0, seed=31, repeat=2, mode="partitioned",
                flags=FLAG_PEER_PUSH)
    res = _run_peer(tmp_path, G, **spec)
    check_steps(res, G, spec)


@pytest.mark.parametrize("G,n", [(2, 2), (4, 4)])
def test_block_over_processes_matches_the_oracle(tmp_path, G, n):
    """The block at world G (E_l = E / G experts per rank, every rank 4 sequences of 128
    tokens), two steps: h, u and out against the oracle block over G ranks, routing by the
    margin rule of _routing_check."""
    from oracle import block as OB
    spec = dict(n_seq=4, S=128, d=256, H=2, f=256, E=8, k=2, cf=1.0, n=n, seed=37, repeat=2, mode="block",
                Ts=[512] * G)
    res = _run_peer(tmp_path, G, **spec)
    for step in range(2):
        sh = S.BlockShape(n_seq=4, seq_len=128, d=256, n_heads=2, f=256, E=8, G=G, k=2, cf=1.0, n_chunks=n)
        ins = [S.gen_block_rank_inputs(37 + step, r, sh, beta=0.5, with_dy=False) for r in range(G)]
        prm = {key: ins[0][key] for key in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "w_qkv", "w_o")}
        ref = OB.block_forward([i["x"] for i in ins], prm, ins[0]["wg"], [i["w1"] for i in ins],
                               [i["w2"] for i in ins], 2, 128, 2, 1.0, n)
        for r in range(G):
            g = res[r]
            assert normwise(g[f"u_s{step}"], ref.u[r]) <= TOL["bf16"]
            assert normwise(g[f"h_s{step}"], ref.h[r]) <= TOL["bf16"]
            rt = ref.moe.routing[r]
            assert int(g[f"C_s{step}"]) == rt.C
            assert np.array_equal(g[f"slot_s{step}"], _admit(g[f"idx_s{step}"], rt.C, sh.E))
            _routing_check(g[f"idx_s{step}"], g[f"slot_s{step}"], rt.logits, rt.idx, rt.slot,
                           g[f"u_s{step}"].astype(np.float64) - ref.u[r], ins[0]["wg"], sh.k)
            same = np.all(g[f"idx_s{step}"] == rt.idx, axis=1) & np.all((g[f"slot_s{step}"] >= 0) == (rt.slot >= 0), axis=1)
            assert same.mean() > 0.95
            assert normwise(g[f"out_s{step}"][same], ref.out[r][same]) <= TOL["bf16"]


def _margin_mask(logits, u, wg, k):
    """Tokens whose top-(k+1) logit margins (oracle side only) exceed an 8-sigma bound of what a
    one-ulp bf16 difference of the gate input u can move: their routing is the same on both
    sides."""
    d = wg.shape[0]
    diff_rms = max(np.sqrt(np.mean((wg[:, a] - wg[:, b]) ** 2))
                   for a in range(wg.shape[1]) for b in range(a + 1, wg.shape[1]))
    du_rms = 2.0 ** -8 * np.sqrt(np.mean(u ** 2))
    bound = 8 * du_rms * np.sqrt(d) * diff_rms
    srt = -np.sort(-logits.astype(np.float64), axis=1)
    kk = min(k + 1, srt.shape[1])
    return np.min(srt[:, :kk - 1] - srt[:, 1:kk], axis=1) > bound


@pytest.mark.parametrize("n_seq,S_,d,H,f,E,k,n,seed", [(4, 256, 256, 2, 512, 4, 2, 2, 11),
                                                        (2, 384, 384, 3, 256, 8, 1, 2, 12),
                                                        (8, 128, 256, 2, 256, 4, 1, 4, 13)])
def test_block_backward_matches_the_oracle(n_seq, S_, d, H, f, E, k, n, seed):
    """lancet_block_backward vs oracle/block.py block_backward: dx, both LayerNorms' gains and
    biases, W_qkv, W_o, Wg, W1, W2 (normwise, bf16 bar).  Capacity not binding (cf = E / k: no
    drops, so a token's routing affects only its own output) and dout = 0 on the tokens whose
    oracle-side top-k margin is within reach of bf16 rounding of the gate input (_margin_mask),
    so every remaining token routes the same way on both sides (checked) and the aggregated
    gradients are comparable."""
    from oracle import block as OB
    cf = E / k
    sh = S.BlockShape(n_seq=n_seq, seq_len=S_, d=d, n_heads=H, f=f, E=E, G=1, k=k, cf=cf, n_chunks=n)
    ins = S.gen_block_rank_inputs(seed, 0, sh, beta=0.5)
    prm = {key: ins[key] for key in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "w_qkv", "w_o")}
    ref = OB.block_forward([ins["x"]], prm, ins["wg"], [ins["w1"]], [ins["w2"]], H, S_, k, cf, n)
    rt = ref.moe.routing[0]
    keep = _margin_mask(rt.logits, ref.u[0], ins["wg"], k)
    dout = S.gen_dy(seed + 1, 0, sh.T, d) * keep[:, None]
    blk = _block(sh, cf_max=cf)
    p = _dev_params(ins)
    blk.forward(to_dev(ins["x"], bf), p, k, cf, n)
    g = blk.backward(to_dev(dout, bf))
    torch.cuda.synchronize()
    assert np.array_equal(blk.debug("idx", sh.T).numpy()[keep], rt.idx[keep])
    assert keep.mean() > 0.75
    rb = OB.block_backward(ref, [ins["x"]], prm, ins["wg"], [ins["w1"]], [ins["w2"]], [dout], H, S_)
    for key in ("dx", "dln1_g", "dln1_b", "dw_qkv", "dw_o", "dln2_g", "dln2_b", "dwg", "dw1", "dw2"):
        got = g[key].float().cpu().numpy()
        e = normwise(got, rb[key][0])
        assert e <= TOL["bf16"], (key, e)
    blk.close()


def test_block_backward_chunk_invariance():
    """The backward of a forward with n = 1 and with n = 4 chunks gives the same input and LN /
    projection gradients bit for bit, the expert weight gradients within fp32 reassociation (the
    merged dW GEMMs see another receive layout)."""
    sh = S.BlockShape(n_seq=4, seq_len=256, d=256, n_heads=2, f=512, E=8, G=1, k=2, cf=1.0, n_chunks=1)
    ins = S.gen_block_rank_inputs(29, 0, sh, beta=0.5)
    dout = to_dev(S.gen_dy(30, 0, sh.T, sh.d), bf)
    res = []
    for n in (1, 4):
        blk = _block(sh)
        p = _dev_params(ins)
        blk.forward(to_dev(ins["x"], bf), p, sh.k, sh.cf, n)
        g = blk.backward(dout)
        torch.cuda.synchronize()
        res.append({key: v.cpu() for key, v in g.items()})
        blk.close()
    for key in ("dx", "dln1_g", "dln1_b", "dw_qkv", "dw_o", "dln2_g", "dln2_b", "dwg"):
        assert torch.equal(res[0][key], res[1][key]), key
    for key in ("dw1", "dw2"):
        assert normwise(res[1][key].numpy(), res[0][key].numpy()) <= 1e-5


@pytest.mark.parametrize("n", [2, 4])
def test_block_stack_pipeline_is_bitwise_consecutive_blocks(n):
    """lancet_block_forward_stack (block l+1's chunk c starts once block l combined chunk c) gives
    every block's output bit for bit as consecutive lancet_block_forward calls, and the stack's
    backward (blocks in reverse, each fed the next one's dx) matches the consecutive one; the
    3-block output is checked against the chained oracle blocks (routing margin rule)."""
    from paper_2404_19429_b200 import block as B
    from oracle import block as OB
    sh = S.BlockShape(n_seq=4, seq_len=256, d=256, n_heads=2, f=512, E=8, G=1, k=2, cf=1.0, n_chunks=n)
    L = 3
    insl = [S.gen_block_rank_inputs(50 + l, 0, sh, beta=0.5) for l in range(L)]
    x = to_dev(insl[0]["x"], bf)
    res = {}
    for mode in ("consecutive", "stack"):
        blks = [_block(sh) for _ in range(L)]
        ps = [_dev_params(i) for i in insl]
        if mode == "stack":
            outs = B.forward_stack(blks, x, ps, sh.k, sh.cf, n)
        else:
            outs, cur = [], x
            for b, p in zip(blks, ps):
                cur = b.forward(cur, p, sh.k, sh.cf, n)
                outs.append(cur)
        dout = to_dev(S.gen_dy(70, 0, sh.T, sh.d), bf)
        grads = []
        for b in reversed(blks):
            g = b.backward(dout)
            grads.append(g)
            dout = g["dx"]
        torch.cuda.synchronize()
        res[mode] = ([o.cpu() for o in outs], [{key: v.cpu() for key, v in g.items()} for g in grads])
        for b in blks:
            b.close()
    for a, b in zip(res["consecutive"][0], res["stack"][0]):
        assert torch.equal(a, b)
    for ga, gb in zip(res["consecutive"][1], res["stack"][1]):
        for key in ga:
            if key in ("dw1", "dw2"):
                assert normwise(gb[key].numpy(), ga[key].numpy()) <= 1e-5
            else:
                assert torch.equal(ga[key], gb[key]), key
    # the chained oracle: each block's oracle on the previous oracle block's output
    cur = insl[0]["x"]
    for l in range(L):
        i = insl[l]
        prm = {key: i[key] for key in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "w_qkv", "w_o")}
        ref = OB.block_forward([cur], prm, i["wg"], [i["w1"]], [i["w2"]], sh.n_heads, sh.seq_len, sh.k, sh.cf, n)
        cur = ref.out[0].astype(np.float32)
    got = res["stack"][0][-1].float().numpy()
    assert normwise(got, cur) <= 3 * TOL["bf16"]
