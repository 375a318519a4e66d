"""GPU parity of the Random gate (R18; LANCET_FLAG_GATE_RANDOM)
against the oracle through the C-ABI: the SplitMix64 draws, slots and counts bit-exact, logits
reported as 0, outputs and gradients within the bf16/fp32 bar, dWg exactly 0."""
import numpy as np
import pytest
import torch

from gpu_harness import TOL, assert_routing_exact, inputs, normwise, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_19429_b200 import build
    build.build()


def _ctx(d, f, E, T, k, seed, dtype="bf16", act="gelu_tanh", extra=0):
    from paper_2404_19429_b200 import FLAG_GATE_RANDOM, lancet
    cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k, max_chunks=8,
                             dtype=dtype, act=act, flags=FLAG_GATE_RANDOM | extra)
    ctx = lancet.Context(cfg)
    ctx.set_gate_seed(seed)
    return ctx


@pytest.mark.parametrize("T,d,E,k,cf,n,seed", [
    (64, 16, 4, 2, 1.25, 2, 0),
    (2500, 256, 8, 2, 0.75, 3, 12345),
    (3001, 96, 64, 4, 1.0, 8, 7),
    (777, 64, 3, 3, 0.5, 5, 2 ** 63 + 5),
    (1, 32, 8, 2, 1.25, 1, 1),
    (513, 32, 1, 1, 1.0, 2, 9),
])
def test_random_gate_routing_bit_exact(T, d, E, k, cf, n, seed):
    ins = inputs(T, d, 8, E, k, seed=T)
    ctx = _ctx(d, 8, E, T, k, seed, act="identity_expert")
    g = run_gpu(ins, E, k, cf, n, act="identity_expert", backward=False, ctx=ctx)
    ctx.close()
    o = run_oracle(ins, k, cf, n, act="identity_expert", backward=False, gate="random", seed=seed)
    assert_routing_exact(g, o)
    assert np.all(g["logits"] == 0)


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_random_gate_forward_backward_parity(dtype):
    T, d, f, E, k, cf, n, seed = 1000, 128, 256, 8, 2, 0.75, 3, 2024
    ins = inputs(T, d, f, E, k, beta=0.5, dtype=dtype, seed=21)
    ctx = _ctx(d, f, E, T, k, seed, dtype=dtype)
    g = run_gpu(ins, E, k, cf, n, dtype=dtype, ctx=ctx)
    ctx.close()
    o = run_oracle(ins, k, cf, n, gate="random", seed=seed)
    assert_routing_exact(g, o)
    assert np.any(o["rt"].slot < 0)
    assert np.all(g["dwg"] == 0)
    for key in ("y", "dx", "dw1", "dw2"):
        assert normwise(g[key], o[key]) <= TOL[dtype], key


def test_random_gate_chunk_invariance_and_seed():
    T, d, f, E, k = 1200, 128, 256, 8, 2
    ins = inputs(T, d, f, E, k, seed=4)
    outs = {}
    for n in (1, 4):
        ctx = _ctx(d, f, E, T, k, 77)
        outs[n] = run_gpu(ins, E, k, 0.75, n, ctx=ctx)
        ctx.close()
    for key in ("y", "dx", "idx", "slot", "dw1", "dw2"):
        assert np.array_equal(outs[1][key], outs[4][key]), key
    ctx = _ctx(d, f, E, T, k, 78)
    other = run_gpu(ins, E, k, 0.75, 1, ctx=ctx, backward=False)
    ctx.close()
    assert not np.array_equal(other["idx"], outs[1]["idx"])


def test_random_gate_excludes_bpr():
    from paper_2404_19429_b200 import FLAG_GATE_BPR, lancet
    ins = inputs(64, 32, 64, 4, 2)
    ctx = _ctx(32, 64, 4, 64, 2, 0, extra=FLAG_GATE_BPR)
    with pytest.raises(lancet.LancetError) as e:
        run_gpu(ins, 4, 2, 1.0, 1, ctx=ctx, backward=False)
    assert e.value.status == 1
    ctx.close()


def test_random_gate_expert_parallel_matches_oracle():
    # two simulated ranks (lancet_local_group), seed 0 on every rank: the draws depend on the
    # rank-local token index only (R18)
    from oracle import moe
    from paper_2404_19429_b200 import FLAG_GATE_RANDOM
    from test_gpu_multirank import make_inputs, oracle_group, run_group
    G, Ts, E, k, n = 2, [700, 513], 8, 2, 3
    ins = make_inputs(G, Ts, 128, 256, E, k, seed=41)
    g = run_group(G, ins, E, k, 0.75, n, flags=FLAG_GATE_RANDOM)
    fwd, b = oracle_group(ins, k, 0.75, n, gate="random")
    sends = [rt.counts for rt in fwd.routing]
    for r in range(G):
        rt = fwd.routing[r]
        assert np.array_equal(g[r]["idx"], rt.idx) and np.array_equal(g[r]["slot"], rt.slot)
        assert np.array_equal(g[r]["recv"], moe.recv_counts(sends, G, r))
        assert np.all(g[r]["dwg"] == 0)
        for key, ref in (("y", fwd.y[r]), ("dx", b["dx"][r]), ("dw1", b["dw1"][r]), ("dw2", b["dw2"][r])):
            assert normwise(g[r][key], ref) <= TOL["bf16"], (r, key)
