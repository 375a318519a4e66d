"""CPU tests of the chunk-count tuner (lancet_tune_chunks, csrc/tuner.cpp): the pipeline
simulation against closed forms, the communication cost model's interpolation and C/n
approximation against the profiles it interpolates, and the profile extraction from timelines."""
import numpy as np
import pytest

from paper_2404_19429_b200.chunk_tuner import N_OPS, OPS, profile_ops, tune

B = 64e6          # bytes of one data exchange at n = 1


def prof(comp_whole=100.0, comm_whole=40.0, once=10.0, fixed=0.0, schedule=0, n=1):
    """Per-chunk op costs at n chunks for whole-batch costs (fixed: per-chunk overhead)."""
    p = np.zeros(N_OPS)
    push_fused = ("GATHER", "K5", "K6")
    for i, k in enumerate(OPS):
        if k in ("GATE", "K7"):
            p[i] = once
        elif k == "COUNTS":
            p[i] = 0.0
        elif k in ("DISPATCH", "COMBINE", "BWD_DISPATCH", "BWD_COMBINE"):
            p[i] = fixed + comm_whole / n
        elif schedule == 1 and k in push_fused:
            p[i] = 0.0
        else:
            p[i] = fixed + comp_whole / n
    return p


def run(schedule=0, **kw):
    profiles = {n: prof(schedule=schedule, n=n, **kw) for n in (1, 2, 4)}
    return tune(profiles, B, schedule, max_chunks=8)


@pytest.mark.parametrize("schedule", [0, 1])
def test_no_communication_is_the_sum_of_compute(schedule):
    best, pred, expo = run(schedule, comm_whole=0.0)
    n_comp = 8 if schedule == 0 else 5            # FC1 FC2 (GATHER K5) DFC2 DFC1 DW (K6)
    # push pipeline: K7 runs on the comm stream beside the dX GEMMs (hidden)
    once = 2 * 10.0 if schedule == 0 else 10.0
    for n in range(1, 9):
        assert pred[n - 1] == pytest.approx(n_comp * 100.0 + once)
        assert expo[n - 1] == pytest.approx(0.0, abs=1e-9)


def test_unchunked_closed_form():
    # n = 1, per-chunk launches: dispatch, combine and the dO exchange sit between producer and
    # consumer; only the dX return hides behind the dW GEMMs
    best, pred, expo = run(0, comp_whole=100.0, comm_whole=40.0)
    assert expo[0] == pytest.approx(3 * 40.0)
    assert pred[0] == pytest.approx(8 * 100.0 + 2 * 10.0 + 3 * 40.0)


def test_chunking_hides_communication_and_fixed_costs_bound_n():
    best, pred, _ = run(0, comp_whole=100.0, comm_whole=40.0)
    assert all(pred[i] > pred[i + 1] for i in range(7))      # no per-chunk cost: more chunks help
    assert best == 8
    best2, pred2, _ = run(0, comp_whole=100.0, comm_whole=40.0, fixed=6.0)
    assert 1 < best2 < 8                                      # per-chunk costs cap n
    assert pred2[best2 - 1] == min(pred2)


def test_comm_model_interpolates_sizes_and_uses_c_over_n():
    # comm profiled at n = 1, 2 only (sizes B, B/2): 100 and 60 us; the model at B/4 extends the
    # segment linearly (20 us per B/4), and a profiled size is reproduced exactly
    comp = prof(comm_whole=0.0, n=1)
    p1, p2 = comp.copy(), prof(comm_whole=0.0, n=2)
    for k in ("DISPATCH", "COMBINE", "BWD_DISPATCH", "BWD_COMBINE"):
        p1[OPS.index(k)] = 100.0
        p2[OPS.index(k)] = 60.0
    _, pred, expo = tune({1: p1, 2: p2}, B, 0, max_chunks=4)
    assert expo[0] == pytest.approx(3 * 100.0)                # n = 1: the profiled 100 us
    # n = 4: per-chunk exchange = model(B/4) = 40 us; four chunks per exchange; mostly hidden
    assert pred[3] < pred[0]


def test_profile_from_timeline():
    tl = [dict(name="expert_fc1", start_us=0.0, end_us=80.0), dict(name="expert_fc1", start_us=100.0, end_us=180.0),
          dict(name="gate", start_us=0.0, end_us=30.0), dict(name="a2a_dispatch_push", start_us=0.0, end_us=10.0),
          dict(name="expert_dw2", start_us=0.0, end_us=50.0), dict(name="expert_dw1", start_us=50.0, end_us=120.0),
          dict(name="expert_fc2", start_us=0.0, end_us=40.0), dict(name="expert_fc2", start_us=20.0, end_us=60.0)]
    p = profile_ops(tl, steps=1, n=2)
    assert p[OPS.index("FC1")] == pytest.approx(80.0)
    assert p[OPS.index("GATE")] == pytest.approx(30.0)
    assert p[OPS.index("DISPATCH")] == pytest.approx(5.0)
    assert p[OPS.index("DW")] == pytest.approx(60.0)
    assert p[OPS.index("FC2")] == pytest.approx(30.0)      # concurrent launches count once (union)


def test_bad_arguments():
    from paper_2404_19429_b200.lancet import LancetError
    with pytest.raises(LancetError):
        tune({1: prof()}, B, 0)                               # one profiled n is not enough
