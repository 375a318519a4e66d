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


def oracle(G, spec):
    import synthetic as S
    from oracle import moe
    ins = []
    for r in range(G):
        sh = S.LayerShape(T=spec["Ts"][r], d=spec["d"], f=spec["f"], E=spec["E"], G=G, k=spec["k"], cf=1.0,
                          n_chunks=1)
        ins.append(S.gen_rank_inputs(spec["seed"], r, sh, beta=spec.get("beta", 0.5)))
    xs = [i["x"] for i in ins]
    act = spec.get("act", "gelu_tanh")
    fwd = moe.forward(xs, ins[0]["wg"], [i["w1"] for i in ins], [i["w2"] for i in ins], spec["k"], spec["cf"],
                      spec["n"], act=act, gate=spec.get("gate", "switch"))
    b = moe.backward(fwd, xs, ins[0]["wg"], [i["w1"] for i in ins], [i["w2"] for i in ins],
                     [i["dy"] for i in ins], act=act)
    return fwd, b


@pytest.mark.parametrize("G,Ts,E,k,n,repeat,act", [
    (2, [700, 513], 8, 2, 3, 1, "gelu_tanh"),       # ragged ranks, 3 chunks
    (2, [600, 600], 4, 1, 1, 2, "gelu_tanh"),       # one chunk, two steps (flag sequence, reuse)
    (4, [300, 420, 256, 333], 8, 2, 4, 2, "gelu_tanh"),
    (2, [500, 450], 4, 2, 2, 2, "identity_expert"), # identity: received rows are the sources back
])
def test_peer_transport_matches_oracle(tmp_path, G, Ts, E, k, n, repeat, act):
    spec = dict(Ts=Ts, d=128, f=256, E=E, k=k, n=n, cf=1.0, seed=40 + G + n, repeat=repeat, act=act)
    res = run_peer(tmp_path, G, **spec)
    fwd, b = oracle(G, spec)
    for r in range(G):
        rt = fwd.routing[r]
        assert np.array_equal(res[r]["idx"], rt.idx) and np.array_equal(res[r]["slot"], rt.slot)
        keys = ("y", "dx", "dwg") + (() if act == "identity_expert" else ("dw1", "dw2"))
        ref = {"y": fwd.y[r], "dx": b["dx"][r], "dwg": b["dwg"][r]}
        if act != "identity_expert":
            ref.update(dw1=b["dw1"][r], dw2=b["dw2"][r])
        for key in keys:
            assert normwise(res[r][key], ref[key]) <= TOL["bf16"], (r, key, normwise(res[r][key], ref[key]))


@pytest.mark.parametrize("gate", ["bpr", "random"])
def test_peer_transport_gate_variants(tmp_path, gate):
    # Batch Prioritized and Random gates over two processes with binding capacity (drops)
    from paper_2404_19429_b200 import FLAG_GATE_BPR, FLAG_GATE_RANDOM
    G = 2
    spec = dict(Ts=[640, 577], d=128, f=256, E=8, k=2, n=3, cf=0.75, seed=77, repeat=2, gate=gate,
                flags=FLAG_GATE_BPR if gate == "bpr" else FLAG_GATE_RANDOM)
    res = run_peer(tmp_path, G, **spec)
    fwd, b = oracle(G, spec)
    for r in range(G):
        rt = fwd.routing[r]
        assert np.any(rt.slot < 0)
        assert np.array_equal(res[r]["idx"], rt.idx) and np.array_equal(res[r]["slot"], rt.slot)
        for key, ref in (("y", fwd.y[r]), ("dx", b["dx"][r]), ("dwg", b["dwg"][r]),
                         ("dw1", b["dw1"][r]), ("dw2", b["dw2"][r])):
            assert normwise(res[r][key], ref) <= TOL["bf16"], (r, key)


@pytest.mark.parametrize("G,Ts,n,act", [(2, [700, 513], 3, "gelu_tanh"), (4, [300, 420, 256, 333], 4, "gelu_tanh"),
                                        (2, [500, 450], 2, "identity_expert")])
def test_peer_push_dispatch_matches_oracle(tmp_path, G, Ts, n, act):
    # LANCET_FLAG_PEER_PUSH across processes: each rank writes its admitted rows into the
    # owners' receive buffers; two steps exercise the receive-buffer-free handshake
    from paper_2404_19429_b200 import FLAG_PEER_PUSH
    spec = dict(Ts=Ts, d=128, f=256, E=8, k=2, n=n, cf=1.0, seed=60 + G + n, repeat=2, act=act,
                flags=FLAG_PEER_PUSH)
    res = run_peer(tmp_path, G, **spec)
    fwd, b = oracle(G, spec)
    for r in range(G):
        rt = fwd.routing[r]
        assert np.array_equal(res[r]["idx"], rt.idx) and np.array_equal(res[r]["slot"], rt.slot)
        keys = ("y", "dx", "dwg") + (() if act == "identity_expert" else ("dw1", "dw2"))
        ref = {"y": fwd.y[r], "dx": b["dx"][r], "dwg": b["dwg"][r]}
        if act != "identity_expert":
            ref.update(dw1=b["dw1"][r], dw2=b["dw2"][r])
        for key in keys:
            assert normwise(res[r][key], ref[key]) <= TOL["bf16"], (r, key)
