"""GPU checks of cross-layer dW scheduling (PAPER.md Opportunity 1 / Alg. 1; R17):
an L-layer stack run with the dW GEMMs moved under other layers' all-to-alls gives bitwise
the same gradients as every layer keeping its own dW (the same kernels on the same data, only
the issue position changes), over the copy-engine transport (one-rank peer group), the NCCL
path (FORCE_EP) and the single-GPU path; plus the ABI's state errors."""
import numpy as np
import pytest
import torch

import synthetic as S
from gpu_harness import TOL, normwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_19429_b200 import build
    build.build()


def make_stack(L, T, d, f, E, k, transport, flags=0):
    from paper_2404_19429_b200 import lancet
    from paper_2404_19429_b200.stack import MoEStack
    cfg = lambda: lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k,  # noqa: E731
                                     max_chunks=8, flags=flags)
    ctxs = [lancet.Context(cfg(), transport=transport) for _ in range(L)]
    params = []
    for l in range(L):
        sh = S.LayerShape(T=T, d=d, f=f, E=E, G=1, k=k, cf=1.0, n_chunks=1)
        ins = S.gen_rank_inputs(100 + l, 0, sh, beta=0.5)
        params.append((torch.from_numpy(ins["wg"]).cuda(),
                       torch.from_numpy(ins["w1"]).cuda().bfloat16(),
                       torch.from_numpy(ins["w2"]).cuda().bfloat16()))
        if l == 0:
            x = torch.from_numpy(ins["x"]).cuda().bfloat16()
            dy = torch.from_numpy(ins["dy"]).cuda().bfloat16()
    return MoEStack(ctxs), params, x, dy


def run(stack, params, x, dy, k, cf, n, plan):
    ys = stack.forward(x, params, k, cf, n)
    grads = [(torch.empty_like(wg), torch.empty(w1.shape, device="cuda"), torch.empty(w2.shape, device="cuda"))
             for wg, w1, w2 in params]
    dxs = stack.backward(dy, grads, plan=plan)
    torch.cuda.synchronize()
    out = [y.float().cpu().numpy() for y in ys] + [dx.float().cpu().numpy() for dx in dxs]
    for g in grads:
        out += [t.cpu().numpy() for t in g]
    return out


# hand plan, L = 3, n = 2 (a2a indices 0..1: dO dispatch, 2..3: dX return):
#   layer 2: dW2 under its own dX return #0, dW1 under layer 1's dO dispatch #0
#   layer 1: dW2 under layer 0's dO dispatch #1, dW1 unassigned (stays after its dX GEMMs)
#   layer 0: dW2 unassigned, dW1 under its own dX return #1
HAND = (np.array([[-1, 0], [0, -1], [2, 1]]), np.array([[-1, 3], [1, -1], [2, 0]]))


@pytest.mark.parametrize("transport,force_ep", [("peer", False), ("nccl", True), ("nccl", False)])
@pytest.mark.parametrize("n", [1, 2])
def test_cross_layer_dw_schedule_is_bitwise_neutral(transport, force_ep, n):
    from paper_2404_19429_b200 import FLAG_FORCE_EP
    from paper_2404_19429_b200.stack import plan_from_costs
    L, T, d, f, E, k, cf = 3, 900, 128, 256, 8, 2, 1.0
    stack, params, x, dy = make_stack(L, T, d, f, E, k, transport, FLAG_FORCE_EP if force_ep else 0)
    ref = run(stack, params, x, dy, k, cf, n, None)
    hl, ha = HAND
    # HAND is written for n = 2: dO dispatch c -> min(c, n-1), dX return 2+c -> n + min(c, n-1)
    ha = np.where(ha < 0, -1, np.where(ha < 2, np.minimum(ha, n - 1), n + np.minimum(ha - 2, n - 1)))
    plans = [(hl, ha), plan_from_costs(np.full((L, 2 * n), 65.0), np.full((L, 2), 230.0))]
    for plan in plans:
        for rep in range(2):                                          # buffers reused across steps
            got = run(stack, params, x, dy, k, cf, n, plan)
            for a, b in zip(got, ref):
                assert np.array_equal(a, b)
    for c in stack.ctxs:
        c.close()


def test_stack_matches_chained_oracle():
    # a 2-layer stack under an Alg. 1 plan against the oracle layers chained through bf16
    from oracle import moe
    from paper_2404_19429_b200.stack import plan_from_costs
    L, T, d, f, E, k, cf, n = 2, 600, 64, 128, 4, 2, 1.0, 2
    stack, params, x, dy = make_stack(L, T, d, f, E, k, "peer")
    plan = plan_from_costs(np.full((L, 2 * n), 65.0), np.full((L, 2), 230.0))
    out = run(stack, params, x, dy, k, cf, n, plan)
    ys, dxs, grads = out[:L], out[L:2 * L], out[2 * L:]
    xin = x.float().cpu().numpy()
    for l in range(L):
        wg, w1, w2 = (t.float().cpu().numpy() for t in params[l])
        fwd = moe.forward([xin], wg, [w1], [w2], k, cf, n)
        assert normwise(ys[l], fwd.y[0]) <= TOL["bf16"]
        dy_l = dy.float().cpu().numpy() if l == L - 1 else dxs[l + 1]
        b = moe.backward(fwd, [xin], wg, [w1], [w2], [dy_l])
        assert normwise(dxs[l], b["dx"][0]) <= TOL["bf16"], l
        for j, key in enumerate(("dwg", "dw1", "dw2")):
            assert normwise(grads[3 * l + j], b[key][0]) <= TOL["bf16"], (l, key)
        xin = ys[l]                                     # the GPU's bf16 output feeds layer l+1
    for c in stack.ctxs:
        c.close()


def test_deferred_dw_state_errors():
    from paper_2404_19429_b200 import FLAG_DEFER_DW, lancet
    stack, params, x, dy = make_stack(1, 256, 64, 128, 4, 2, "nccl")
    ctx = stack.ctxs[0]
    wg, w1, w2 = params[0]
    with pytest.raises(lancet.LancetError) as e:
        ctx.backward_dw(3)                                   # nothing pending
    assert e.value.status == 5
    ctx.set_flags(FLAG_DEFER_DW)
    ctx.forward(x, wg, w1, w2, 2, 1.0, 1)
    dx, dwg, dw1, dw2 = ctx.backward(dy)
    with pytest.raises(lancet.LancetError) as e:
        ctx.forward(x, wg, w1, w2, 2, 1.0, 1)                # dW still pending
    assert e.value.status == 5
    ctx.backward_dw(2)
    with pytest.raises(lancet.LancetError):
        ctx.backward_dw(2)                                   # already enqueued
    ctx.backward_dw(1)
    torch.cuda.synchronize()
    ctx.set_flags(0)
    ref = [t.clone() for t in (dx, dwg, dw1, dw2)]
    ctx.forward(x, wg, w1, w2, 2, 1.0, 1)
    got = ctx.backward(dy)
    torch.cuda.synchronize()
    for a, b in zip(got, ref):
        assert torch.equal(a, b)
    ctx.close()
