"""The library's native dW schedule pass (lancet_dw_schedule / lancet_stack_dw_plan, host C++,
no device) against the oracle (oracle/dw_schedule.py) -- CPU only."""
import random

import numpy as np

from oracle import dw_schedule as D
from paper_2404_19429_b200 import lancet


def _oracle_assign(kinds, cost, edges):
    asg = D.greedy_assign(kinds, cost, D.label_overlappable(kinds, edges))
    out = np.full(len(kinds), -1, dtype=np.int32)
    for i, a in asg.items():
        out[i] = a
    return out


def test_native_matches_oracle_on_random_dags():
    r = random.Random(3)
    for trial in range(200):
        n = r.randint(2, 40)
        edges = [(i, j) for i in range(n) for j in range(i + 1, n) if r.random() < 0.12]
        kinds = [r.choice([D.OTHER, D.A2A, D.DW, D.DW]) for _ in range(n)]
        # integer-valued costs make exact ties (the lowest-index rule) frequent
        cost = [float(r.randint(1, 12)) for _ in range(n)]
        got = lancet.dw_schedule(kinds, cost, edges)
        assert np.array_equal(got, _oracle_assign(kinds, cost, edges)), trial


def test_native_spec_hand_traces():
    assert lancet.dw_schedule([1, 2, 2, 2], [100, 60, 90, 30], []).tolist() == [-1, -1, 0, 0]
    assert lancet.dw_schedule([1, 1, 2, 2], [100, 100, 100, 100], []).tolist() == [-1, -1, 0, 1]
    # a dW fed by the all-to-all is never eligible for it
    assert lancet.dw_schedule([1, 2], [100, 50], [(0, 1)]).tolist() == [-1, -1]


def test_native_stack_plan_matches_oracle():
    r = random.Random(9)
    for trial in range(60):
        L, n = r.randint(1, 5), r.randint(1, 4)
        t_a2a = np.array([[float(r.randint(20, 120)) for _ in range(2 * n)] for _ in range(L)])
        t_dw = np.array([[float(r.randint(50, 250)) for _ in range(2)] for _ in range(L)])
        hl, ha = lancet.stack_dw_plan(t_a2a, t_dw)
        kinds, names, edges, idx = D.stack_backward_program(L, n)
        cost = [0.0] * len(kinds)
        for l in range(L):
            for c in range(n):
                cost[idx[("B1", l, c)]] = t_a2a[l, c]
                cost[idx[("B2", l, c)]] = t_a2a[l, n + c]
            cost[idx[("DW2", l, 0)]] = t_dw[l, 0]
            cost[idx[("DW1", l, 0)]] = t_dw[l, 1]
        asg = D.greedy_assign(kinds, cost, D.label_overlappable(kinds, edges))
        where = {}
        for (name, l, c), i in idx.items():
            if name in ("B1", "B2"):
                where[i] = (l, c if name == "B1" else n + c)
        for l in range(L):
            for w, name in ((0, "DW2"), (1, "DW1")):
                i = idx[(name, l, 0)]
                want = where[asg[i]] if i in asg else (-1, -1)
                assert (hl[l, w], ha[l, w]) == want, (trial, l, name)
                if hl[l, w] >= 0:
                    assert hl[l, w] <= l                      # never before its own backward


def test_native_stack_plan_hand_trace():
    # the hand trace of tests/test_oracle_dw_schedule.py::test_stack_greedy_hand_trace
    hl, ha = lancet.stack_dw_plan([[65.0, 65.0], [65.0, 65.0]], [[230.0, 230.0], [230.0, 230.0]])
    assert hl.tolist() == [[0, -1], [1, 0]]
    assert ha.tolist() == [[1, -1], [1, 0]]


def test_native_schedule_argument_errors():
    import pytest
    with pytest.raises(lancet.LancetError) as e:
        lancet.dw_schedule([1, 2], [10.0, 5.0], [(0, 7)])          # edge to a missing instruction
    assert e.value.status == 1
    with pytest.raises(lancet.LancetError):
        lancet.stack_dw_plan(np.zeros((0, 2)), np.zeros((0, 2)))     # no layers
