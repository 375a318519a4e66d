"""GPU tests of the push mode of the peer transport (LANCET_FLAG_PEER_PUSH) on a one-rank peer
group: the device-built exchange plan and the kernel flags make the step free of host
synchronisation, so it can be captured in a CUDA graph; the fused exchange kernels run on the
comm stream beside the expert GEMMs; the failure paths (abort, fixed flags) hold."""
import numpy as np
import pytest
import torch

from gpu_harness import TOL, inputs, normwise, run_gpu, run_oracle, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_19429_b200 import build
    build.build()


def _push_ctx(T, d, f, E, k, flags=0, act="gelu_tanh"):
    from paper_2404_19429_b200 import FLAG_PEER_PUSH, lancet
    cfg = lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k, max_chunks=8, act=act,
                             flags=FLAG_PEER_PUSH | flags)
    return lancet.Context(cfg, transport="peer")


@pytest.mark.parametrize("n,act,launches", [(4, "gelu_tanh", False), (1, "gelu_tanh", False),
                                            (3, "identity_expert", False), (4, "gelu_tanh", True)])
def test_push_step_replays_from_a_cuda_graph(n, act, launches):
    # capture one fwd+bwd step into a CUDA graph, then replay it on new inputs copied into the
    # captured buffers: every output equals an eager step on the same inputs bit for bit
    # (launches: the per-chunk-launch schedule instead of the device-side GEMM pipeline)
    from paper_2404_19429_b200 import FLAG_CHUNK_LAUNCHES
    T, d, f, E, k, cf = 2048, 256, 512, 8, 2, 1.0
    ctx = _push_ctx(T, d, f, E, k, act=act, flags=FLAG_CHUNK_LAUNCHES if launches else 0)
    ins = [inputs(T, d, f, E, k, beta=0.5, seed=300 + i) for i in range(3)]
    bf = torch.bfloat16
    x = to_dev(ins[0]["x"], bf)
    wg = to_dev(ins[0]["wg"], torch.float32)
    w1 = to_dev(ins[0]["w1"], bf)
    w2 = to_dev(ins[0]["w2"], bf)
    dy = to_dev(ins[0]["dy"], bf)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    dwg = torch.empty(wg.shape, device="cuda")
    dw1 = torch.empty(w1.shape, device="cuda") if act != "identity_expert" else None
    dw2 = torch.empty(w2.shape, device="cuda") if act != "identity_expert" else None
    idx = torch.empty(T, k, dtype=torch.int32, device="cuda")

    def step(stream=None):
        _, ix, _, _ = ctx.forward(x, wg, w1, w2, k, cf, n, y=y, stream=stream)
        ctx.backward(dy, dx=dx, dwg=dwg, dw1=dw1, dw2=dw2, stream=stream)
        idx.copy_(ix)

    def load(i):
        for t, key in ((x, "x"), (wg, "wg"), (w1, "w1"), (w2, "w2"), (dy, "dy")):
            t.copy_(to_dev(ins[i][key], t.dtype))

    def snap():
        torch.cuda.synchronize()
        out = dict(y=y.clone(), dx=dx.clone(), dwg=dwg.clone(), idx=idx.clone())
        if dw1 is not None:
            out.update(dw1=dw1.clone(), dw2=dw2.clone())
        return out

    eager = {}
    for i in (1, 2):
        load(i)
        step()
        eager[i] = snap()
    load(0)
    step()                                   # warm-up (function attributes, tensor maps)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            step(stream=s)
    torch.cuda.current_stream().wait_stream(s)
    for i in (1, 2, 1):
        load(i)
        g.replay()
        got = snap()
        for key, ref in eager[i].items():
            assert torch.equal(got[key], ref), (i, key)
    o = run_oracle(ins[2], k, cf, n, act=act)
    load(2)
    g.replay()
    got = snap()
    for key in ("y", "dx", "dwg"):
        assert normwise(got[key].float().cpu().numpy(), o[key]) <= TOL["bf16"], key
    ctx.close()


@pytest.mark.parametrize("launches", [False, True])
def test_push_exchanges_overlap_the_expert_gemms(launches):
    # the fused exchange kernels run on the comm stream, on the SMs the persistent GEMMs leave
    # free.  Device-side pipeline (default): chunk c >= 1's dispatch runs under fc1 (one launch
    # over all chunks, waiting per chunk on the device), chunk c's combine under chunk c+1's fc2,
    # chunk c's dX return under chunk c+1's dfc1 or the merged dW GEMMs.
    # Per-chunk launches: chunk c's combine under chunk c+1's GEMMs, its dX return under its dW.
    from paper_2404_19429_b200 import FLAG_CHUNK_LAUNCHES, FLAG_TIMELINE
    T, d, f, E, k, n = 16384, 1024, 4096, 8, 2, 4
    ctx = _push_ctx(T, d, f, E, k, flags=FLAG_TIMELINE | (FLAG_CHUNK_LAUNCHES if launches else 0))
    ins = inputs(T, d, f, E, k, beta=0.25, seed=4)
    for _ in range(3):
        run_gpu(ins, E, k, 1.25, n, ctx=ctx)
    tl = ctx.timeline()
    ctx.close()

    def span(name, ch):
        r = [o for o in tl if o["name"] == name and o["chunk"] == ch]
        assert r, (name, ch)
        return r[0]["start_us"], r[0]["end_us"]

    def overlap(a, b):
        return max(0.0, min(a[1], b[1]) - max(a[0], b[0]))

    if launches:
        fwd = [overlap(span("a2a_combine_fused", ch), (span("expert_fc1", ch + 1)[0], span("expert_fc2", ch + 1)[1]))
               for ch in range(n - 1)]
        bwd = [overlap(span("a2a_bwd_combine_fused", ch), (span("expert_dw2", ch)[0], span("expert_dw1", ch)[1]))
               for ch in range(n)]
    else:
        fc1, dw1 = span("expert_fc1", -1), span("expert_dw1", -1)
        fwd = [overlap(span("a2a_dispatch_push", ch), fc1) for ch in range(1, n)] + \
              [overlap(span("a2a_combine_fused", ch), span("expert_fc2", ch + 1)) for ch in range(n - 1)]
        bwd = [overlap(span("a2a_bwd_combine_fused", ch), (span("expert_dfc1", ch + 1)[0] if ch + 1 < n else
                                                           span("expert_dw2", -1)[0], dw1[1])) for ch in range(n)]
    assert sum(o > 0 for o in fwd) >= n - 2, fwd
    assert sum(o > 0 for o in bwd) >= n - 1, bwd
    for name in ("a2a_dispatch_push", "a2a_combine_fused", "a2a_bwd_dispatch_push", "a2a_bwd_combine_fused"):
        ops = [o for o in tl if o["name"] == name]
        assert len(ops) == n and all(o["lane"] == 1 for o in ops), name


def test_push_mode_is_fixed_at_creation_and_abort_poisons():
    from paper_2404_19429_b200 import lancet
    T, d, f, E, k, n = 1000, 128, 256, 8, 2, 2
    ins = inputs(T, d, f, E, k, beta=0.5, seed=12)
    ctx = _push_ctx(T, d, f, E, k)
    ref = run_gpu(ins, E, k, 1.0, n, ctx=ctx)
    ctx.set_flags(0)                           # PEER_PUSH cannot be switched off: kept
    got = run_gpu(ins, E, k, 1.0, n, ctx=ctx)
    for key in ("y", "dx", "dwg", "dw1", "dw2"):
        assert np.array_equal(got[key], ref[key]), key
    ctx.status()
    ctx.peer_abort()
    with pytest.raises(lancet.LancetError) as e:
        run_gpu(ins, E, k, 1.0, n, ctx=ctx)
    assert e.value.status == 5 and "abort" in str(e.value)
    ctx.close()


def test_no_comm_timing_variant_runs():
    # LANCET_FLAG_NO_COMM (timing only): same ops minus the exchanges; must run and finish
    from paper_2404_19429_b200 import FLAG_NO_COMM
    T, d, f, E, k, n = 1000, 128, 256, 8, 2, 2
    ins = inputs(T, d, f, E, k, beta=0.5, seed=12)
    ctx = _push_ctx(T, d, f, E, k, flags=FLAG_NO_COMM)
    run_gpu(ins, E, k, 1.0, n, ctx=ctx)
    run_gpu(ins, E, k, 1.0, n, ctx=ctx)
    ctx.status()
    ctx.close()
