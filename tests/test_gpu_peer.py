"""GPU parity of the copy-engine peer transport (lancet_create_peer): G processes (torchrun),
all on GPU 0 -- CUDA IPC works between processes of one device -- each a rank of the
expert-parallel layer; the all-to-alls are cudaMemcpyAsync pulls from the peers' mapped
buffers, ordered by stream wait-value / write-value flags.  Checked against the oracle."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from gpu_harness import TOL, normwise

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2404_19429_b200 import build
    build.build()


def run_peer(tmp_path, G, **spec):
    spec = dict(spec)
    env = dict(os.environ, PEER_SPEC=json.dumps(spec), PEER_OUT=str(tmp_path))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + (os.getpid() % 1000)),
           os.path.join(ROOT, "tests", "peer_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [dict(np.load(os.path.join(tmp_path, f"rank{i}.npz"))) for i in range(G)]


def oracle(G, spec, step=0):
    """The oracle layer on the inputs of step `step` (seed + step, as peer_worker.py)."""
    import synthetic as S
    from oracle import moe
    ins = []
    for r in range(G):
        sh = S.LayerShape(T=spec["Ts"][r], d=spec["d"], f=spec["f"], E=spec["E"], G=G, k=spec["k"], cf=1.0,
                          n_chunks=1)
        ins.append(S.gen_rank_inputs(spec["seed"] + step, r, sh, beta=spec.get("beta", 0.5)))
    xs = [i["x"] for i in ins]
    act = spec.get("act", "gelu_tanh")
    fwd = moe.forward(xs, ins[0]["wg"], [i["w1"] for i in ins], [i["w2"] for i in ins], spec["k"], spec["cf"],
                      spec["n"], act=act, gate=spec.get("gate", "switch"))
    b = moe.backward(fwd, xs, ins[0]["wg"], [i["w1"] for i in ins], [i["w2"] for i in ins],
                     [i["dy"] for i in ins], act=act)
    return fwd, b


def check_steps(res, G, spec, keys=("y", "dx", "dwg", "dw1", "dw2")):
    """Every step of every rank against the oracle of that step's inputs."""
    for step in range(spec.get("repeat", 1)):
        fwd, b = oracle(G, spec, step)
        for r in range(G):
            rt = fwd.routing[r]
            assert np.array_equal(res[r][f"idx_s{step}"], rt.idx) and np.array_equal(res[r][f"slot_s{step}"], rt.slot)
            ref = {"y": fwd.y[r], "dx": b["dx"][r], "dwg": b["dwg"][r]}
            if "dw1" in b:
                ref.update(dw1=b["dw1"][r], dw2=b["dw2"][r])
            for key in keys:
                if key not in ref:
                    continue
                e = normwise(res[r][f"{key}_s{step}"], ref[key])
                assert e <= TOL["bf16"], (step, r, key, e)


@pytest.mark.parametrize("G,Ts,E,k,n,repeat,act", [
    (2, [700, 513], 8, 2, 3, 1, "gelu_tanh"),       # ragged ranks, 3 chunks
    (2, [600, 600], 4, 1, 1, 2, "gelu_tanh"),       # one chunk, two steps (flag sequence, reuse)
    (4, [300, 420, 256, 333], 8, 2, 4, 2, "gelu_tanh"),
    (2, [500, 450], 4, 2, 2, 2, "identity_expert"), # identity: received rows are the sources back
])
def test_peer_transport_matches_oracle(tmp_path, G, Ts, E, k, n, repeat, act):
    spec = dict(Ts=Ts, d=128, f=256, E=E, k=k, n=n, cf=1.0, seed=40 + G + n, repeat=repeat, act=act)
    res = run_peer(tmp_path, G, **spec)
    check_steps(res, G, spec)


@pytest.mark.parametrize("gate", ["bpr", "random"])
def test_peer_transport_gate_variants(tmp_path, gate):
    # Batch Prioritized and Random gates over two processes with binding capacity (drops)
    from paper_2404_19429_b200 import FLAG_GATE_BPR, FLAG_GATE_RANDOM
    G = 2
    spec = dict(Ts=[640, 577], d=128, f=256, E=8, k=2, n=3, cf=0.75, seed=77, repeat=2, gate=gate,
                flags=FLAG_GATE_BPR if gate == "bpr" else FLAG_GATE_RANDOM)
    res = run_peer(tmp_path, G, **spec)
    fwd, _ = oracle(G, spec)
    assert all(np.any(rt.slot < 0) for rt in fwd.routing)
    check_steps(res, G, spec)


@pytest.mark.parametrize("G,Ts,n,act", [(2, [700, 513], 3, "gelu_tanh"), (4, [300, 420, 256, 333], 4, "gelu_tanh"),
                                        (2, [500, 450], 2, "identity_expert")])
def test_peer_push_dispatch_matches_oracle(tmp_path, G, Ts, n, act):
    # LANCET_FLAG_PEER_PUSH across processes: each rank writes its admitted rows into the
    # owners' receive buffers; two steps exercise the receive-buffer-free handshake
    from paper_2404_19429_b200 import FLAG_PEER_PUSH
    spec = dict(Ts=Ts, d=128, f=256, E=8, k=2, n=n, cf=1.0, seed=60 + G + n, repeat=2, act=act,
                flags=FLAG_PEER_PUSH)
    res = run_peer(tmp_path, G, **spec)
    check_steps(res, G, spec)


@pytest.mark.parametrize("push", [True, False])
def test_eight_processes_at_the_configs1_layer_shape(tmp_path, push):
    # the layout of the 8-GPU run (G = 8, E = 8 so E_l = 1, d = 1024, f = 4096, top-2, n = 4) as
    # 8 processes sharing one GPU, T = 2048 per rank, two steps with different inputs: routing
    # bit-exact on every rank, y / dx on 64 sampled tokens per rank, dW1 / dW2 of two ranks'
    # experts in full (all their rows from all 8 sources), against the oracle
    from paper_2404_19429_b200 import FLAG_PEER_PUSH
    G, T = 8, 2048
    rng = np.random.default_rng(8)
    sample = [sorted(rng.choice(T, 64, replace=False).tolist()) for _ in range(G)]
    spec = dict(Ts=[T] * G, d=1024, f=4096, E=8, k=2, n=4, cf=1.25, seed=800 + push, repeat=2, beta=0.25,
                flags=FLAG_PEER_PUSH if push else 0, sample=sample)
    res = run_peer(tmp_path, G, **spec)
    from oracle import moe
    import synthetic as S
    for step in range(2):
        ins = []
        for r in range(G):
            sh = S.LayerShape(T=T, d=1024, f=4096, E=8, G=G, k=2, cf=1.0, n_chunks=1)
            ins.append(S.gen_rank_inputs(spec["seed"] + step, r, sh, beta=0.25))
        xs, wg = [i["x"] for i in ins], ins[0]["wg"]
        w1, w2, dys = [i["w1"] for i in ins], [i["w2"] for i in ins], [i["dy"] for i in ins]
        # y / dx on the sampled tokens (all experts), dW1 / dW2 of every expert on all its rows
        fs = moe.forward(xs, wg, w1, w2, 2, 1.25, 4, token_subset=sample)
        bs = moe.backward(fs, xs, wg, w1, w2, dys)
        for r in range(G):
            rt = fs.routing[r]
            assert np.array_equal(res[r][f"idx_s{step}"], rt.idx), (step, r)
            assert np.array_equal(res[r][f"slot_s{step}"], rt.slot), (step, r)
            tok = np.asarray(sample[r])
            for key, ref in (("y", fs.y[r][tok]), ("dx", bs["dx"][r][tok])):
                e = normwise(res[r][f"{key}_s{step}"], ref)
                assert e <= TOL["bf16"], (step, r, key, e)
        for r in (0, 5):
            fe = moe.forward(xs, wg, w1, w2, 2, 1.25, 4, experts=[r])
            be = moe.backward(fe, xs, wg, w1, w2, dys)
            for key in ("dw1", "dw2"):
                e = normwise(res[r][f"{key}_s{step}"][0], be[key][r][0])
                assert e <= TOL["bf16"], (step, r, key, e)


def test_peer_wait_times_out_and_poisons(tmp_path):
    # rank 1 never runs its step: rank 0's push-mode waits give up after the timeout instead of
    # hanging, and its context reports which flag never came
    from paper_2404_19429_b200 import FLAG_PEER_PUSH
    spec = dict(Ts=[256, 256], d=128, f=256, E=4, k=2, n=2, cf=1.0, seed=3, mode="timeout", timeout_ms=1500,
                flags=FLAG_PEER_PUSH)
    res = run_peer(tmp_path, 2, **spec)
    msg = str(res[0]["msg"])
    assert "ERR_STATE" in msg and "timed out" in msg and "rank 1" in msg, msg


def test_peer_config_mismatch_is_refused(tmp_path):
    # ranks created with different max_tokens: import fails on every rank (no silent overflow of
    # the smaller receive buffer, no mismatched flag slots)
    spec = dict(Ts=[256, 256], d=128, f=256, E=4, k=2, n=2, cf=1.0, seed=3, mode="mismatch")
    res = run_peer(tmp_path, 2, **spec)
    for r in range(2):
        assert "import failed" in str(res[r]["msg"]), str(res[r]["msg"])
