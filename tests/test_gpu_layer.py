"""GPU parity of the MoE layer step (single rank) against the oracle, through the C-ABI.

Sizes span several tiles of every kernel (gate blocks of 64 tokens, 256-token scan tiles,
128-row GEMM tiles) with ragged tails; BASELINE.json configs[1] (the bench workload) is
checked at full size on sampled outputs."""
import numpy as np
import pytest

import torch

from gpu_harness import (TOL, assert_routing_exact, inputs, normwise, run_gpu, run_oracle)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_19429_b200 import build
    build.build()


@pytest.mark.parametrize("T,d,E,k,beta,cf,n", [
    (64, 16, 4, 2, 0.5, 1.25, 2),          # BASELINE configs[0] per-rank shape, 64 tokens
    (2500, 256, 8, 2, 0.5, 1.25, 3),       # 10 scan tiles, ragged
    (3001, 96, 64, 4, 1.0, 1.0, 8),        # many experts, k=4, drops
    (777, 64, 3, 1, 0.0, 0.5, 5),          # odd E, top-1, capacity binding hard
    (1, 32, 8, 2, 0.5, 1.25, 1),           # single token
    (513, 32, 1, 1, 0.0, 1.0, 2),          # one expert
    (1500, 192, 32, 2, 0.5, 1.25, 3),      # warp-streaming gate, 8 threads per token
    (999, 320, 16, 3, 0.5, 1.0, 2),        # warp-streaming gate, 4 threads per token, ragged
    (10001, 256, 8, 2, 0.5, 1.25, 4),      # two tokens per thread (T >= 9472), ragged last warp
    (9473, 192, 16, 3, 0.5, 1.0, 3),       # two tokens per thread at E = 16, one token past a block
])
def test_routing_bit_exact(T, d, E, k, beta, cf, n):
    ins = inputs(T, d, 8, E, k, beta=beta, seed=T)
    g = run_gpu(ins, E, k, cf, n, act="identity_expert", backward=False)
    o = run_oracle(ins, k, cf, n, act="identity_expert", backward=False)
    assert_routing_exact(g, o)


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("act", ["gelu_tanh", "relu"])
def test_forward_backward_parity(dtype, act):
    # d % 64 == 0, E = 8: the warp-streaming gate (bf16 and fp32 x); general K6/K7 (d % 256 != 0)
    T, d, f, E, k, cf, n = 1000, 128, 256, 8, 2, 1.0, 3
    ins = inputs(T, d, f, E, k, beta=0.5, dtype=dtype, seed=11)
    g = run_gpu(ins, E, k, cf, n, dtype=dtype, act=act)
    o = run_oracle(ins, k, cf, n, act=act)
    assert_routing_exact(g, o)
    assert np.any(o["rt"].slot < 0), "case must exercise drops"
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        err = normwise(g[key], o[key])
        assert err <= TOL[dtype], (key, err)


def test_identity_experts_reproduce_gate_weighted_inputs():
    T, d, E, k = 1500, 64, 8, 2
    ins = inputs(T, d, 8, E, k, beta=1.0, seed=5)
    g = run_gpu(ins, E, k, 0.75, 4, act="identity_expert")
    o = run_oracle(ins, k, 0.75, 4, act="identity_expert")
    assert_routing_exact(g, o)
    scale = np.where(g["slot"] >= 0, g["w"], 0.0).sum(1, dtype=np.float64)
    want = scale[:, None] * ins["x"].astype(np.float64)
    # one fp32 fma chain + one bf16 rounding: within 1 bf16 ulp (2^-8 relative)
    assert np.all(np.abs(g["y"] - want) <= 2.0 ** -8 * np.abs(want) + 1e-30)
    for key in ("y", "dx", "dwg"):
        assert normwise(g[key], o[key]) <= TOL["bf16"], key


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_chunk_count_does_not_change_results(dtype):
    # capacity passing: chunked routing == unchunked routing, so every output is identical
    T, d, f, E, k = 1200, 128, 256, 8, 2
    ins = inputs(T, d, f, E, k, beta=0.5, dtype=dtype, seed=3)
    ref = run_gpu(ins, E, k, 1.0, 1, dtype=dtype)
    for n in (2, 4, 8):
        g = run_gpu(ins, E, k, 1.0, n, dtype=dtype)
        for key in ("y", "dx", "idx", "slot", "dw1", "dw2", "dwg"):
            assert np.array_equal(g[key], ref[key]), (n, key)
        assert np.array_equal(g["send"].sum(1), ref["send"][:, 0])


def test_renormalized_weights():
    from paper_2404_19429_b200 import FLAG_RENORMALIZE
    T, d, f, E, k = 700, 64, 128, 8, 2
    ins = inputs(T, d, f, E, k, beta=0.5, seed=9)
    g = run_gpu(ins, E, k, 1.0, 2, flags=FLAG_RENORMALIZE)
    o = run_oracle(ins, k, 1.0, 2, renorm=True)
    assert np.allclose(g["w"].sum(1), 1.0, atol=1e-6)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        assert normwise(g[key], o[key]) <= TOL["bf16"], key


def test_api_errors_on_device():
    import torch
    from paper_2404_19429_b200 import lancet
    cfg = lancet.LayerConfig(d_model=64, d_ffn=128, n_experts=4, max_tokens=32, max_k=2)
    ctx = lancet.Context(cfg)
    dy = torch.zeros(32, 64, dtype=torch.bfloat16, device="cuda")
    ctx._last = (dy, dy, dy, dy)
    with pytest.raises(lancet.LancetError) as e:
        ctx.backward(dy)
    assert e.value.status == 5                                   # ERR_STATE
    ins = inputs(32, 64, 128, 4, 2)
    x = torch.from_numpy(ins["x"]).cuda().bfloat16()
    wg = torch.from_numpy(ins["wg"]).cuda()
    w1 = torch.from_numpy(ins["w1"]).cuda().bfloat16()
    w2 = torch.from_numpy(ins["w2"]).cuda().bfloat16()
    for kw in (dict(k=3, cf=1.0, n=1), dict(k=2, cf=0.0, n=1), dict(k=2, cf=1.0, n=9)):
        with pytest.raises(lancet.LancetError) as e:
            ctx.forward(x, wg, w1, w2, kw["k"], kw["cf"], kw["n"])
        assert e.value.status == 1                               # ERR_ARG
    ctx.close()


def test_full_size_gpt_moe_layer():
    # BASELINE.json configs[1] per GPU: T=16384, d=1024, f=4096, E=8, top-2, bf16; n=4 chunks --
    # the whole layer against the whole oracle (fwd + bwd, ~1.7 TFLOP of fp64 on the host)
    T, d, f, E, k, cf, n = 16384, 1024, 4096, 8, 2, 1.25, 4
    ins = inputs(T, d, f, E, k, beta=0.25, seed=2024)
    g = run_gpu(ins, E, k, cf, n)
    o = run_oracle(ins, k, cf, n)
    assert_routing_exact(g, o)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        err = normwise(g[key], o[key])
        assert err <= TOL["bf16"], (key, err)
    dropped = np.all(g["slot"] < 0, axis=1)
    assert np.all(g["y"][dropped] == 0)


def test_full_size_fp32_mode():
    # the fp32 mode (north_star: <= 1e-5 against the oracle) at the configs[1] per-GPU shape:
    # fp32 x / W1 / W2 through the SIMT GEMMs, the fp32 gate and every fp32 kernel variant
    T, d, f, E, k, cf, n = 16384, 1024, 4096, 8, 2, 1.25, 4
    ins = inputs(T, d, f, E, k, beta=0.25, dtype="fp32", seed=2025)
    g = run_gpu(ins, E, k, cf, n, dtype="fp32")
    o = run_oracle(ins, k, cf, n)
    assert_routing_exact(g, o)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        err = normwise(g[key], o[key])
        assert err <= TOL["fp32"], (key, err)


@pytest.mark.parametrize("k", [1, 2, 4])
def test_switch_gate_ties_break_to_the_lower_expert(k):
    # duplicated Wg columns give bitwise-equal logits (R1: the same fp32 chain): top-k must order
    # the tied experts by index (R2), on the GPU as in the oracle; capacity binding so the tie
    # order also decides the slots and the drops
    T, d, f, E, n = 1500, 128, 256, 8, 3
    ins = inputs(T, d, f, E, k, beta=0.5, seed=77 + k)
    wg = ins["wg"].copy()
    wg[:, 5] = wg[:, 2]
    wg[:, 7] = wg[:, 2]
    wg[:, 4] = wg[:, 1]
    ins["wg"] = wg
    g = run_gpu(ins, E, k, 0.8, n)
    o = run_oracle(ins, k, 0.8, n)
    assert_routing_exact(g, o)
    tied = np.isin(o["rt"].idx, [1, 2, 4, 5, 7])
    assert tied.mean() > 0.2, "the case must route many tokens to the tied experts"
    assert np.any(o["rt"].slot < 0)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        assert normwise(g[key], o[key]) <= TOL["bf16"], key


@pytest.mark.parametrize("T,d,f,E,k,n", [
    (1000, 128, 256, 8, 2, 3),        # BN=128 (fc2/dfc1 N=d=128) and BN=256 (fc1 N=f=256)
    (2300, 256, 512, 4, 2, 2),        # K = 256 / 512: several k-blocks per tile, ring wraps
    (300, 128, 384, 2, 1, 1),         # N = 384: BN=128 x 3 n-tiles; tiny groups
    (900, 64, 96, 8, 2, 2),           # ragged: N and K below one tile (TMA zero-fill / clipping)
    (700, 200, 136, 4, 2, 3),         # ragged N, K and dW M (d, f not multiples of 64 / 128)
    (1200, 72, 264, 16, 2, 1),        # ragged, pair tiles for dW M = 264 not a multiple of 256
])
def test_tcgen05_gemm_matches_simt_gemm(T, d, f, E, k, n):
    # the tcgen05/TMA path and the SIMT path compute the same fp32-accumulated GEMMs;
    # they may differ only by accumulation order -> far below the bf16 tolerance
    from paper_2404_19429_b200 import FLAG_SIMT_GEMM
    ins = inputs(T, d, f, E, k, beta=0.5, seed=T + d)
    tc = run_gpu(ins, E, k, 1.0, n)
    simt = run_gpu(ins, E, k, 1.0, n, flags=FLAG_SIMT_GEMM)
    for key in ("idx", "slot"):
        assert np.array_equal(tc[key], simt[key])
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        # two accumulation orders may round a bf16 output 1 ulp apart (2^-8 relative)
        assert normwise(tc[key], simt[key]) <= 2 * 2.0 ** -8, (key, normwise(tc[key], simt[key]))
    o = run_oracle(ins, k, 1.0, n)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        assert normwise(tc[key], o[key]) <= TOL["bf16"], key


@pytest.mark.parametrize("E,k", [(16, 2), (4, 1), (8, 4)])
def test_gate_backward_paths(E, k):
    # d % 256 != 0: the general K6 (Wg^T in shared memory) and K7 (partials over 64-token
    # tiles) kernels, for E <= 8 and E > 8
    T, d, f = 900, 128, 256
    ins = inputs(T, d, f, E, k, beta=0.5, seed=E * 10 + k)
    g = run_gpu(ins, E, k, 1.0, 3)
    o = run_oracle(ins, k, 1.0, 3)
    assert_routing_exact(g, o)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        assert normwise(g[key], o[key]) <= TOL["bf16"], key


@pytest.mark.parametrize("T,d,E,k,dtype", [
    (1999, 256, 8, 2, "bf16"),      # the GPT-MoE path shape class: E <= 8, d % 256 == 0
    (1531, 512, 5, 1, "fp32"),      # odd E (padded to 8 in registers), top-1, fp32 storage
    (2048, 256, 3, 3, "bf16"),      # k = 3 (ring slot sized for KK = 4), E padded to 4
    (700, 2048, 2, 2, "bf16"),      # widest streamed row: 256 threads x 8 dims
    (37, 256, 8, 2, "fp32"),        # fewer tokens than blocks
    (1500, 256, 16, 2, "bf16"),     # wide: 2 lanes per dim group
    (1200, 512, 32, 1, "fp32"),     # wide: 4 lanes per dim group, d split over 2 blocks
    (900, 1024, 64, 4, "bf16"),     # wide: 8 lanes per dim group, d split over 4 blocks, k = 4
    (333, 256, 64, 3, "bf16"),      # wide, k = 3, ragged
])
def test_gate_backward_streaming_paths(T, d, E, k, dtype):
    # E <= 8, d % 256 == 0, d <= 2048: K6 with Wg^T in registers and K7 partials over
    # contiguous token ranges, both fed by per-thread cp.async rings
    f = 256
    ins = inputs(T, d, f, E, k, beta=0.5, dtype=dtype, seed=T + E)
    g = run_gpu(ins, E, k, 1.0, 2, dtype=dtype)
    o = run_oracle(ins, k, 1.0, 2)
    assert_routing_exact(g, o)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        err = normwise(g[key], o[key])
        assert err <= TOL[dtype], (key, err)


@pytest.mark.parametrize("T,d,f,E,k", [
    (3000, 256, 512, 4, 2),         # fc1 / dfc2 / dW2: 2 N tiles of 256 -> one multicast pair
    (2100, 512, 1024, 2, 2),        # 4 / 2 N tiles; few, large groups
])
def test_gemm_multicast_is_bitwise_neutral(T, d, f, E, k):
    # two CTA pairs sharing an A tile by TMA multicast issue the same MMAs in the same K order
    # as one pair alone: every output must be bitwise identical
    from paper_2404_19429_b200 import FLAG_GEMM_MULTICAST
    ins = inputs(T, d, f, E, k, beta=0.5, seed=T)
    mc = run_gpu(ins, E, k, 1.25, 2, flags=FLAG_GEMM_MULTICAST)
    one = run_gpu(ins, E, k, 1.25, 2)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        assert np.array_equal(mc[key], one[key]), key
    o = run_oracle(ins, k, 1.25, 2)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        assert normwise(mc[key], o[key]) <= TOL["bf16"], key


@pytest.mark.parametrize("T,d,E,k,dtype", [
    (3001, 256, 8, 2, "bf16"),
    (1400, 512, 6, 1, "fp32"),
    (900, 1024, 4, 4, "bf16"),
])
def test_fused_gate_backward_matches_two_kernel_path(T, d, E, k, dtype):
    # world 1: K6 + K7 in one pass vs the two streaming kernels.  dx is the same arithmetic
    # (row sum in j order, then the gate term in e order): bitwise.  dWg partials cover other
    # token ranges: fp32 reassociation only.
    from paper_2404_19429_b200 import FLAG_UNFUSED_GATE_BWD, FLAG_NO_SIDE_STREAM
    f = 256
    ins = inputs(T, d, f, E, k, beta=0.5, dtype=dtype, seed=T + d)
    fu = run_gpu(ins, E, k, 1.0, 2, dtype=dtype, flags=FLAG_NO_SIDE_STREAM)
    un = run_gpu(ins, E, k, 1.0, 2, dtype=dtype, flags=FLAG_NO_SIDE_STREAM | FLAG_UNFUSED_GATE_BWD)
    side = run_gpu(ins, E, k, 1.0, 2, dtype=dtype)
    assert np.array_equal(side["dx"], un["dx"]) and np.array_equal(side["dwg"], un["dwg"])
    assert np.array_equal(fu["dx"], un["dx"])
    assert normwise(fu["dwg"], un["dwg"]) <= 1e-6
    o = run_oracle(ins, k, 1.0, 2)
    for key in ("dx", "dwg"):
        assert normwise(fu[key], o[key]) <= TOL[dtype], key


@pytest.mark.parametrize("n,act,transport", [(1, "gelu_tanh", "nccl"), (4, "gelu_tanh", "nccl"),
                                             (3, "identity_expert", "nccl"), (4, "gelu_tanh", "peer"),
                                             (2, "identity_expert", "peer")])
def test_force_ep_nccl_path_matches_single_gpu_path(n, act, transport):
    # the expert-parallel path (counts exchange, per-chunk grouped NCCL send/recv over a
    # one-rank communicator, S1/S2 chunk scheduler, per-chunk expert GEMMs) on one GPU: rows are
    # independent and K orders equal, so y / dx / routing are bitwise those of the single-GPU
    # path; dW accumulates per chunk (fp32 reassociation)
    from paper_2404_19429_b200 import FLAG_FORCE_EP
    T, d, f, E, k = 2000, 256, 512, 8, 2
    ins = inputs(T, d, f, E, k, beta=0.5, seed=77 + n)
    # "peer": the copy-engine transport over a one-rank peer group (self pulls)
    ep = run_gpu(ins, E, k, 1.0, n, act=act, flags=FLAG_FORCE_EP if transport == "nccl" else 0,
                 transport=transport)
    one = run_gpu(ins, E, k, 1.0, n, act=act)
    for key in ("idx", "slot", "y", "dx"):
        assert np.array_equal(ep[key], one[key]), key
    keys = ("dwg",) if act == "identity_expert" else ("dwg", "dw1", "dw2")
    for key in keys:
        assert normwise(ep[key], one[key]) <= 1e-5, key
    o = run_oracle(ins, k, 1.0, n, act=act)
    for key in ("y", "dx") + keys:
        assert normwise(ep[key], o[key]) <= TOL["bf16"], key


def test_programmatic_dependent_launch_is_bitwise_neutral():
    # PDL lets a kernel start while its predecessor drains; every kernel waits before touching
    # memory, so the results must be bitwise those of plain stream ordering
    from paper_2404_19429_b200 import FLAG_NO_PDL
    T, d, f, E, k = 2500, 256, 512, 8, 2
    ins = inputs(T, d, f, E, k, beta=0.5, seed=31)
    a = run_gpu(ins, E, k, 1.0, 2)
    b = run_gpu(ins, E, k, 1.0, 2, flags=FLAG_NO_PDL)
    for key in ("idx", "slot", "y", "dx", "dwg", "dw1", "dw2"):
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_force_ep_renormalized_and_fp32(dtype):
    # the NCCL path with renormalised combine weights, and with fp32 storage (SIMT GEMMs)
    from paper_2404_19429_b200 import FLAG_FORCE_EP, FLAG_RENORMALIZE
    T, d, f, E, k = 1100, 128, 256, 4, 2
    ins = inputs(T, d, f, E, k, beta=0.5, dtype=dtype, seed=5)
    g = run_gpu(ins, E, k, 1.0, 3, dtype=dtype, flags=FLAG_FORCE_EP | FLAG_RENORMALIZE)
    o = run_oracle(ins, k, 1.0, 3, renorm=True)
    assert_routing_exact(g, o)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        assert normwise(g[key], o[key]) <= TOL[dtype], key


def test_context_reuse_across_shapes_and_chunk_counts():
    # one context, successive steps with different T and n: each equals a fresh context's run
    from paper_2404_19429_b200 import lancet
    d, f, E, k = 256, 512, 8, 2
    cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=3000, max_k=k, max_chunks=8)
    ctx = lancet.Context(cfg)
    for T, n in ((3000, 4), (1234, 1), (2999, 8), (64, 2)):
        ins = inputs(T, d, f, E, k, beta=0.5, seed=T)
        a = run_gpu(ins, E, k, 1.0, n, ctx=ctx)
        b = run_gpu(ins, E, k, 1.0, n, max_tokens=3000)
        for key in ("idx", "slot", "y", "dx", "dwg", "dw1", "dw2"):
            assert np.array_equal(a[key], b[key]), (T, n, key)
    ctx.close()


def test_peer_context_requires_import():
    # the peer transport refuses to run before its peers are mapped (ERR_STATE, nothing enqueued)
    import ctypes
    from paper_2404_19429_b200 import lancet
    lib = lancet.load_library()
    cfg = lancet.LayerConfig(d_model=128, d_ffn=256, n_experts=4, max_tokens=256, max_k=2)
    p = ctypes.c_void_p()
    assert lib.lancet_create_peer(ctypes.byref(p), 1, 0, 0, ctypes.byref(cfg._c())) == 0
    x = torch.zeros(256, 128, dtype=torch.bfloat16, device="cuda")
    wg = torch.zeros(128, 4, device="cuda")
    w1 = torch.zeros(4, 256, 128, dtype=torch.bfloat16, device="cuda")
    w2 = torch.zeros(4, 128, 256, dtype=torch.bfloat16, device="cuda")
    y = torch.empty_like(x)
    st = lib.lancet_moe_forward(p, x.data_ptr(), wg.data_ptr(), w1.data_ptr(), w2.data_ptr(), 256, 2,
                                ctypes.c_double(1.0), 2, y.data_ptr(), None, None, None, None)
    assert st == 5                                               # ERR_STATE
    assert lib.lancet_destroy(p) == 0


@pytest.mark.parametrize("E", [32, 64])
def test_large_token_count_gate_backward(E):
    # T = 64k with many experts: the streaming K6/K7 stage per-block dlogit rows in shared
    # memory, which must be split over more blocks at this size (a launch once failed here);
    # identity experts keep the oracle cheap (routing, y, dx, dWg against it)
    T, d, k, cf, n = 65536, 1024, 2, 1.25, 4
    ins = inputs(T, d, 8, E, k, beta=0.25, seed=64)
    g = run_gpu(ins, E, k, cf, n, act="identity_expert")
    o = run_oracle(ins, k, cf, n, act="identity_expert")
    assert_routing_exact(g, o)
    for key in ("y", "dx", "dwg"):
        assert normwise(g[key], o[key]) <= TOL["bf16"], key


@pytest.mark.parametrize("T,E,k", [(4097, 32, 1), (2053, 16, 1), (3001, 32, 3)])
def test_gate_backward_odd_tokens_per_block(T, E, k):
    # the wide / streaming K6 stage an odd number of (tokens x choices) row ids in front of the
    # dlogit rows they read as float2: the dlogit staging is 16-byte aligned (an odd count once
    # faulted at E = 32, k = 1, d = 2048 -- found by compute-sanitizer on the block backward)
    d = 2048
    ins = inputs(T, d, 8, E, k, beta=0.25, seed=65)
    g = run_gpu(ins, E, k, 1.0, 2, act="identity_expert")
    o = run_oracle(ins, k, 1.0, 2, act="identity_expert")
    assert_routing_exact(g, o)
    for key in ("y", "dx", "dwg"):
        assert normwise(g[key], o[key]) <= TOL["bf16"], key


@pytest.mark.parametrize("n,act,serial", [(1, "gelu_tanh", False), (3, "gelu_tanh", False),
                                          (2, "identity_expert", False), (4, "gelu_tanh", True),
                                          (3, "identity_expert", True)])
def test_push_dispatch_is_bitwise_the_pull_path(n, act, serial):
    # LANCET_FLAG_PEER_PUSH: permute fused with the dispatch exchange (rows written straight into
    # the owner's receive buffer) over a one-rank peer group: same rows at the same positions,
    # so every output equals the copy-engine pull path bit for bit; two steps (buffer reuse)
    from paper_2404_19429_b200 import FLAG_PEER_PUSH, FLAG_SERIAL, lancet
    T, d, f, E, k = 2000, 256, 512, 8, 2
    ins = inputs(T, d, f, E, k, beta=0.5, seed=91 + n)
    outs = {}
    sf = FLAG_SERIAL if serial else 0        # serial baseline: chunks merged into one group
    for name, fl in (("pull", sf), ("push", FLAG_PEER_PUSH | sf)):
        cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k, max_chunks=8,
                                 act=act, flags=fl)
        ctx = lancet.Context(cfg, transport="peer")
        run_gpu(ins, E, k, 1.0, n, act=act, ctx=ctx)
        outs[name] = run_gpu(ins, E, k, 1.0, n, act=act, ctx=ctx)
        ctx.close()
    keys = ("idx", "slot", "y", "dx", "dwg") + (() if act == "identity_expert" else ("dw1", "dw2"))
    for key in keys:
        if key in ("dw1", "dw2") and n > 1 and not serial:
            # the push pipeline merges the chunks' dW GEMMs (one K range per expert): fp32
            # reassociation against the per-chunk reduce-add of the pull path
            assert normwise(outs["push"][key], outs["pull"][key]) <= 1e-5, key
            continue
        assert np.array_equal(outs["push"][key], outs["pull"][key]), key
    o = run_oracle(ins, k, 1.0, n, act=act)
    for key in ("y", "dx"):
        assert normwise(outs["push"][key], o[key]) <= TOL["bf16"], key


def test_push_forward_without_backward_releases_the_outputs():
    # with the fused combine, K4 and K5 read the owners' expert outputs in place and K5 releases
    # them; a forward that is not followed by a backward must release them at the next forward
    # (no stall), and the step after it is unchanged
    from paper_2404_19429_b200 import FLAG_PEER_PUSH, lancet
    T, d, f, E, k, n = 1000, 128, 256, 8, 2, 2
    ins = inputs(T, d, f, E, k, beta=0.5, seed=5)
    cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k, max_chunks=8,
                             flags=FLAG_PEER_PUSH)
    ctx = lancet.Context(cfg, transport="peer")
    ref = run_gpu(ins, E, k, 1.0, n, ctx=ctx)
    run_gpu(ins, E, k, 1.0, n, ctx=ctx, backward=False)          # forward only
    run_gpu(ins, E, k, 1.0, n, ctx=ctx, backward=False)          # and again
    got = run_gpu(ins, E, k, 1.0, n, ctx=ctx)
    ctx.close()
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        assert np.array_equal(got[key], ref[key]), key


@pytest.mark.parametrize("E,n,transport", [(192, 1, "local"), (256, 2, "local"), (136, 1, "peer")])
def test_more_than_128_gemm_groups(E, n, transport):
    # the tcgen05 kernel caches 128 group entries: larger group tables (E > 128 at world 1, or
    # n * E_l > 128 on the expert-parallel path) run as several launches -- same results as the
    # SIMT GEMM and the oracle, never a silent fallback
    from paper_2404_19429_b200 import FLAG_SIMT_GEMM, lancet
    T, d, f, k = 3000, 128, 256, 2
    ins = inputs(T, d, f, E, k, beta=0.5, seed=E + n)
    if transport == "peer":
        mk = lambda fl: lancet.Context(lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k,
                                                          max_chunks=8, flags=fl), transport="peer")
        c1, c2 = mk(0), mk(FLAG_SIMT_GEMM)
        tc = run_gpu(ins, E, k, 1.0, n, ctx=c1)
        simt = run_gpu(ins, E, k, 1.0, n, ctx=c2)
        c1.close()
        c2.close()
    else:
        tc = run_gpu(ins, E, k, 1.0, n)
        simt = run_gpu(ins, E, k, 1.0, n, flags=FLAG_SIMT_GEMM)
    assert tc["launches"][0] > simt["launches"][0], "the group table must have been split"
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        assert normwise(tc[key], simt[key]) <= 2 * 2.0 ** -8, key
    o = run_oracle(ins, k, 1.0, n)
    for key in ("y", "dx", "dw1", "dw2"):
        assert normwise(tc[key], o[key]) <= TOL["bf16"], key


def test_misaligned_pointers_are_refused():
    from paper_2404_19429_b200 import lancet
    T, d, f, E, k = 64, 64, 128, 4, 2
    cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k)
    ctx = lancet.Context(cfg)
    ins = inputs(T, d, f, E, k)
    flat = torch.zeros(T * d + 8, dtype=torch.bfloat16, device="cuda")
    x = flat[1:1 + T * d].view(T, d)                     # 2-byte offset
    x.copy_(torch.from_numpy(ins["x"]).cuda().bfloat16())
    wg = torch.from_numpy(ins["wg"]).cuda()
    w1 = torch.from_numpy(ins["w1"]).cuda().bfloat16()
    w2 = torch.from_numpy(ins["w2"]).cuda().bfloat16()
    with pytest.raises(lancet.LancetError) as e:
        ctx.forward(x, wg, w1, w2, k, 1.0, 1)
    assert e.value.status == 1 and "aligned" in str(e.value)
    ctx.close()


def test_nccl_registered_buffers_are_bitwise_neutral(monkeypatch):
    # the NCCL data plane with its buffers from ncclMemAlloc registered with the communicator
    # (user-buffer registration) against plain cudaMalloc buffers (LANCET_NCCL_REGISTER=0): the
    # exchanges move the same bytes, so two steps on new inputs agree bit for bit
    from paper_2404_19429_b200 import FLAG_FORCE_EP, lancet
    T, d, f, E, k, n = 1500, 256, 512, 8, 2, 3
    outs, regs = [], []
    for env in ("1", "0"):
        monkeypatch.setenv("LANCET_NCCL_REGISTER", env)
        cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k, max_chunks=8,
                                 flags=FLAG_FORCE_EP)
        ctx = lancet.Context(cfg)
        try:
            steps = [run_gpu(inputs(T, d, f, E, k, beta=0.5, seed=500 + s), E, k, 1.0, n, ctx=ctx)
                     for s in range(2)]
            regs.append(ctx.nccl_registered())
        finally:
            ctx.close()
        outs.append(steps)
    assert regs[1] == 0
    print("registered buffers:", regs[0])
    for a, b in zip(*outs):
        for key in ("idx", "slot", "y", "dx", "dwg", "dw1", "dw2"):
            assert np.array_equal(a[key], b[key]), key


def test_maximum_experts_and_top_k():
    # the API's upper limits at once: E = 256 experts (kMaxExperts: tiled gate with 8 experts x 4
    # tokens per thread, 256-row scan histograms, > 128 GEMM groups in batched launches) and
    # k = 8 (kMaxK) with a binding capacity, against the oracle
    T, d, f, E, k, cf, n = 3000, 64, 128, 256, 8, 1.25, 4
    ins = inputs(T, d, f, E, k, beta=0.5, seed=256)
    g = run_gpu(ins, E, k, cf, n)
    o = run_oracle(ins, k, cf, n)
    assert_routing_exact(g, o)
    assert np.any(o["rt"].slot < 0), "case must exercise drops"
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        err = normwise(g[key], o[key])
        assert err <= TOL["bf16"], (key, err)


def test_maximum_chunk_count_expert_parallel_path():
    # n = 64 chunks (kMaxChunks) on the expert-parallel path (one-rank NCCL communicator): 64
    # per-chunk exchanges and GEMM groups of ~4 rows per expert; rows are independent, so y / dx
    # / routing are bitwise the single-GPU path's and the gradients meet the oracle
    from paper_2404_19429_b200 import FLAG_FORCE_EP, lancet
    T, d, f, E, k, cf, n = 2000, 128, 256, 8, 2, 1.0, 64
    ins = inputs(T, d, f, E, k, beta=0.5, seed=64)
    cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k, max_chunks=64,
                             flags=FLAG_FORCE_EP)
    ctx = lancet.Context(cfg)
    try:
        ep = run_gpu(ins, E, k, cf, n, ctx=ctx)
    finally:
        ctx.close()
    one = run_gpu(ins, E, k, cf, 1)                 # the single-GPU path is unchunked
    for key in ("idx", "slot", "y", "dx"):
        assert np.array_equal(ep[key], one[key]), key
    o = run_oracle(ins, k, cf, n)
    assert_routing_exact(ep, o)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        err = normwise(ep[key], o[key])
        assert err <= TOL["bf16"], (key, err)


@pytest.mark.parametrize("path", ["single", "force_ep", "push"])
def test_experts_that_receive_no_rows(path):
    # degenerate routing: two experts are never selected (their Wg columns are pushed far below
    # the others), so their GEMM groups are empty on every chunk -- their weight gradients must
    # be exactly zero, everything else must meet the oracle, on the single-GPU path, the
    # expert-parallel NCCL path and the push pipeline (one-rank peer group)
    from paper_2404_19429_b200 import FLAG_FORCE_EP, FLAG_PEER_PUSH, lancet
    T, d, f, E, k, cf, n = 1300, 128, 256, 8, 2, 1.25, 3
    ins = inputs(T, d, f, E, k, beta=0.5, seed=13)
    ins["wg"][:, 3] = -ins["wg"][:, 3].__abs__() - 0.5
    ins["wg"][:, 6] = -ins["wg"][:, 6].__abs__() - 0.5
    ins["x"] = np.abs(ins["x"]).astype(ins["x"].dtype)          # x >= 0: those logits stay lowest
    o = run_oracle(ins, k, cf, n)
    assert not np.isin(o["rt"].idx, [3, 6]).any(), "construction must leave experts 3 and 6 unused"
    if path == "single":
        g = run_gpu(ins, E, k, cf, n)
    else:
        fl = FLAG_FORCE_EP if path == "force_ep" else FLAG_PEER_PUSH
        cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k, max_chunks=8, flags=fl)
        ctx = lancet.Context(cfg, transport="nccl" if path == "force_ep" else "peer")
        try:
            g = run_gpu(ins, E, k, cf, n, ctx=ctx)
        finally:
            ctx.close()
    assert_routing_exact(g, o)
    for e in (3, 6):
        assert not np.any(g["dw1"][e]) and not np.any(g["dw2"][e]), e
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        err = normwise(g[key], o[key])
        assert err <= TOL["bf16"], (key, err)
