"""GPU parity of Batch Prioritized Routing (R16;
LANCET_FLAG_GATE_BPR) against the oracle, through the C-ABI: routing (idx, slot, counts)
bit-exact -- the fp64 importance score decides who is dropped, evaluated in fp64 on both
sides -- and outputs/gradients within the bf16/fp32 bar.  Ties (duplicated tokens, identical
scores) go to the lower token index on both sides."""
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


def _bpr():
    from paper_2404_19429_b200 import FLAG_GATE_BPR
    return FLAG_GATE_BPR


@pytest.mark.parametrize("T,d,E,k,beta,cf,n", [
    (64, 16, 4, 2, 0.5, 1.25, 2),          # BASELINE configs[0] per-rank shape
    (2500, 256, 8, 2, 0.5, 1.25, 3),       # 10 scan tiles, ragged
    (3001, 96, 64, 4, 1.0, 1.0, 8),        # many experts, k=4
    (777, 64, 3, 1, 1.0, 0.5, 5),          # odd E, top-1, capacity binding hard
    (1, 32, 8, 2, 0.5, 1.25, 1),           # single token
    (513, 32, 1, 1, 0.0, 0.5, 2),          # one expert: BPR keeps the top half by score
    (5000, 128, 16, 2, 1.0, 0.25, 4),      # most pairs dropped: deep radix select
])
def test_bpr_routing_bit_exact(T, d, E, k, beta, cf, n):
    ins = inputs(T, d, 8, E, k, beta=beta, seed=T + 17)
    g = run_gpu(ins, E, k, cf, n, act="identity_expert", backward=False, flags=_bpr())
    o = run_oracle(ins, k, cf, n, act="identity_expert", backward=False, gate="bpr")
    assert_routing_exact(g, o)
    if cf < 1.0 and T > 1 and E > 1:
        # BPR must differ from token-major admission somewhere in these binding cases
        sw = run_oracle(ins, k, cf, n, act="identity_expert", backward=False)
        assert not np.array_equal(sw["rt"].slot, o["rt"].slot)


def test_bpr_ties_go_to_lower_token():
    # 37 distinct rows repeated: every score occurs ~54 times, so the radix select ends on a
    # tie group that the capacity splits
    T, d, E, k = 2000, 64, 4, 2
    ins = inputs(T, d, 8, E, k, beta=0.5, seed=77)
    ins["x"] = np.ascontiguousarray(ins["x"][np.arange(T) % 37])
    g = run_gpu(ins, E, k, 0.5, 3, act="identity_expert", backward=False, flags=_bpr())
    o = run_oracle(ins, k, 0.5, 3, act="identity_expert", backward=False, gate="bpr")
    assert np.any(o["rt"].slot < 0)
    assert_routing_exact(g, o)


def test_bpr_nonbinding_capacity_equals_switch():
    T, d, E, k = 1500, 64, 8, 2
    ins = inputs(T, d, 8, E, k, beta=0.0, seed=5)
    a = run_gpu(ins, E, k, 8.0, 2, act="identity_expert", backward=False, flags=_bpr())
    b = run_gpu(ins, E, k, 8.0, 2, act="identity_expert", backward=False)
    assert np.all(a["slot"] >= 0)
    for key in ("idx", "slot", "y", "send"):
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_bpr_forward_backward_parity(dtype):
    T, d, f, E, k, cf, n = 1000, 128, 256, 8, 2, 0.75, 3
    ins = inputs(T, d, f, E, k, beta=0.5, dtype=dtype, seed=21)
    g = run_gpu(ins, E, k, cf, n, dtype=dtype, flags=_bpr())
    o = run_oracle(ins, k, cf, n, gate="bpr")
    assert_routing_exact(g, o)
    assert np.any(o["rt"].slot < 0), "case must exercise drops"
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        err = normwise(g[key], o[key])
        assert err <= TOL[dtype], (key, err)


def test_bpr_chunk_count_does_not_change_results():
    # partition after the gate (fig:part_after_gate): chunked == unchunked, bitwise
    T, d, f, E, k = 1200, 128, 256, 8, 2
    ins = inputs(T, d, f, E, k, beta=0.5, seed=4)
    ref = run_gpu(ins, E, k, 0.75, 1, flags=_bpr())
    for n in (2, 4, 8):
        g = run_gpu(ins, E, k, 0.75, n, flags=_bpr())
        for key in ("y", "dx", "idx", "slot", "dw1", "dw2", "dwg"):
            assert np.array_equal(g[key], ref[key]), (n, key)


def test_bpr_full_size_gpt_moe_layer_sampled():
    # BASELINE.json configs[1] per GPU with the Batch Prioritized gate
    T, d, f, E, k, cf, n = 16384, 1024, 4096, 8, 2, 1.25, 4
    ins = inputs(T, d, f, E, k, beta=0.25, seed=2025)
    g = run_gpu(ins, E, k, cf, n, flags=_bpr())
    rng = np.random.default_rng(1)
    sub = np.sort(np.concatenate([rng.choice(T, 48, replace=False), [0, T - 1]]))
    o = run_oracle(ins, k, cf, n, token_subset=[sub], gate="bpr")
    assert np.any(o["rt"].slot < 0)
    assert_routing_exact(g, o)
    assert normwise(g["y"][sub], o["y"][sub]) <= TOL["bf16"]
    assert normwise(g["dx"][sub], o["dx"][sub]) <= TOL["bf16"]


def test_bpr_expert_parallel_matches_oracle():
    from test_gpu_multirank import make_inputs, oracle_group, run_group
    from oracle import moe
    G, Ts, E, k, n = 2, [700, 513], 8, 2, 3
    ins = make_inputs(G, Ts, 128, 256, E, k, seed=31)
    g = run_group(G, ins, E, k, 0.75, n, flags=_bpr())
    fwd, b = oracle_group(ins, k, 0.75, n, gate="bpr")
    sends = [rt.counts for rt in fwd.routing]
    for r in range(G):
        rt = fwd.routing[r]
        assert np.array_equal(g[r]["idx"], rt.idx) and np.array_equal(g[r]["slot"], rt.slot)
        assert np.array_equal(g[r]["send"], rt.counts)
        assert np.array_equal(g[r]["recv"], moe.recv_counts(sends, G, r))
        for key, ref in (("y", fwd.y[r]), ("dx", b["dx"][r]), ("dw1", b["dw1"][r]), ("dw2", b["dw2"][r])):
            assert normwise(g[r][key], ref) <= TOL["bf16"], (r, key)
