"""Host logic of the stack executor (paper_2404_19429_b200/stack.py) without a device: which
context defers its dW GEMMs and which filler slots each backward receives for a plan
(R17), checked with stand-in contexts that record the calls."""
import numpy as np

from paper_2404_19429_b200 import FLAG_DEFER_DW
from paper_2404_19429_b200.stack import WHICH, MoEStack


class FakeCfg:
    def __init__(self):
        self.flags = 0


class FakeCtx:
    def __init__(self, name, log):
        self.name, self.log, self.cfg = name, log, FakeCfg()

    def set_flags(self, f):
        self.cfg.flags = f
        self.log.append(("flags", self.name, f))

    def set_dw_fillers(self, fl):
        self.log.append(("fillers", self.name, [(o.name, w, a) for o, w, a in fl]))

    def backward(self, dy, dwg=None, dw1=None, dw2=None, stream=None):
        self.log.append(("backward", self.name, self.cfg.flags))
        return f"dx{self.name}", None, None, None


def _run(plan, L=3, n=2):
    log = []
    ctxs = [FakeCtx(l, log) for l in range(L)]
    st = MoEStack(ctxs)
    st.n = n
    dxs = st.backward("dy", [(None, None, None)] * L, plan=plan)
    return log, dxs


def test_no_plan_keeps_every_layer_on_its_own_schedule():
    log, dxs = _run(None)
    assert [e[1] for e in log if e[0] == "backward"] == [2, 1, 0]          # backward order
    assert all(e[2] == [] for e in log if e[0] == "fillers")
    assert all(not (e[2] & FLAG_DEFER_DW) for e in log if e[0] == "backward")
    assert dxs == ["dx0", "dx1", "dx2"]


def test_plan_maps_to_fillers_and_deferral():
    n = 2
    hl = np.array([[-1, 0], [0, -1], [2, 1]])      # [layer][part]: part 0 = dW2, 1 = dW1
    ha = np.array([[-1, 3], [1, -1], [2, 0]])
    log, _ = _run((hl, ha), n=n)
    fills = {e[1]: e[2] for e in log if e[0] == "fillers"}
    deferred = {e[1] for e in log if e[0] == "backward" and e[2] & FLAG_DEFER_DW}
    assert deferred == {0, 1, 2}
    # layer 2 carries its own dW2 under its dX return #0 (index n + 0 = 2)
    assert fills[2] == [(2, WHICH[0], 2)]
    # layer 1 carries layer 2's dW1 under its dO dispatch #0, and its own unassigned dW1 stays
    # after its dX GEMMs (index n)
    assert sorted(fills[1]) == sorted([(2, WHICH[1], 0), (1, WHICH[1], n)])
    # layer 0 carries layer 1's dW2 (dispatch #1), its own dW1 (return #1) and its own
    # unassigned dW2 (index n)
    assert sorted(fills[0]) == sorted([(1, WHICH[0], 1), (0, WHICH[1], 3), (0, WHICH[0], n)])
    # flags restored after the backward
    assert all(not (c & FLAG_DEFER_DW) for c in [e[2] for e in log if e[0] == "flags"][-3:])


def test_layers_without_assignment_are_not_deferred():
    hl = np.array([[-1, -1], [1, 1]])
    ha = np.array([[-1, -1], [2, 3]])
    log, _ = _run((hl, ha), L=2)
    deferred = {e[1] for e in log if e[0] == "backward" and e[2] & FLAG_DEFER_DW}
    assert deferred == {1}
