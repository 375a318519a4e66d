"""CPU tests of the chunk-count tuner (paper_2404_19429_b200/chunk_tuner.py): the two-lane
simulation against closed forms, and the cost-model fit against the model it inverts."""
import pytest

from paper_2404_19429_b200.chunk_tuner import CHUNKED, ONCE, CostModel, OpModel, best_n, fit, simulate

COMM = ("a2a_counts", "a2a_dispatch", "a2a_combine", "a2a_bwd_dispatch", "a2a_bwd_combine")


def model(comp_whole=100.0, comm_whole=50.0, fixed=0.0, once=10.0):
    m = CostModel()
    for name in CHUNKED:
        m.chunked[name] = OpModel(fixed, comm_whole if name.startswith("a2a") else comp_whole)
    for name in ONCE:
        m.once[name] = 0.0 if name == "a2a_counts" else once
    return m


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_no_communication_is_the_sum_of_compute(n):
    m = model(comm_whole=0.0)
    r = simulate(m, n)
    n_chunked_comp = sum(1 for x in CHUNKED if not x.startswith("a2a"))
    assert r["step_us"] == pytest.approx(n_chunked_comp * 100.0 + 3 * 10.0)
    assert r["exposed_comm_us"] == pytest.approx(0.0)


def test_unchunked_and_serial_closed_forms():
    m = model(comp_whole=100.0, comm_whole=40.0)
    compute = 9 * 100.0 + 3 * 10.0               # 9 chunked compute ops + gate, permute, K7
    # n = 1: dispatch, combine and the first backward exchange sit between producer and
    # consumer; only the second backward exchange hides behind the dW GEMMs
    r = simulate(m, 1)
    assert r["exposed_comm_us"] == pytest.approx(3 * 40.0)
    assert r["step_us"] == pytest.approx(compute + 3 * 40.0)
    # one lane (the unoverlapped baseline): everything adds up
    s = simulate(m, 4, serial=True)
    assert s["exposed_comm_us"] == pytest.approx(4 * 40.0 + 0.0)
    assert s["step_us"] == pytest.approx(compute + 4 * 40.0)


def test_chunking_hides_communication_and_fixed_costs_bound_n():
    m = model(comp_whole=100.0, comm_whole=40.0)
    t = {n: simulate(m, n)["step_us"] for n in (1, 2, 4, 8)}
    assert t[1] > t[2] > t[4] > t[8]              # no per-chunk cost: more chunks always help
    m2 = model(comp_whole=100.0, comm_whole=40.0, fixed=2.0)
    n_best, preds = best_n(m2)
    assert n_best == 2                           # per-chunk costs cap n (n <= 4)
    assert all(p["step_us"] >= preds[1]["step_us"] for p in preds)


def test_fit_recovers_the_model():
    true = model(comp_whole=120.0, comm_whole=60.0, fixed=3.0)
    lines = {}
    for n in (1, 4):
        k = {name: {"us": true.chunked[name].per_chunk(n) * n} for name in CHUNKED}
        k.update({name: {"us": v} for name, v in true.once.items()})
        lines[n] = {"kernels": k, "launch_groups": {name: n for name in CHUNKED}}
    m = fit(lines)
    for name in CHUNKED:
        assert m.chunked[name].fixed == pytest.approx(3.0)
        assert m.chunked[name].whole == pytest.approx(true.chunked[name].whole)
    for n in (2, 8):
        assert simulate(m, n)["step_us"] == pytest.approx(simulate(true, n)["step_us"])
