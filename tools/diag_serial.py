"""Diagnostic: determinism of the pipelined world>1 schedule vs the serial one (local group)."""
import sys
import numpy as np
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from test_gpu_multirank import make_inputs, run_group
from paper_2404_19429_b200 import FLAG_SERIAL

G, E, k, n = 2, 8, 2, 4
ins = make_inputs(G, [900, 800], 128, 256, E, k, seed=9)
a = run_group(G, ins, E, k, 1.0, n)
a2 = run_group(G, ins, E, k, 1.0, n)
b = run_group(G, ins, E, k, 1.0, n, flags=FLAG_SERIAL)
b2 = run_group(G, ins, E, k, 1.0, n, flags=FLAG_SERIAL)
for r in range(G):
    for key in ("y", "dx"):
        for name, u, v in (("a-a2", a, a2), ("b-b2", b, b2), ("a-b", a, b)):
            dif = u[r][key] != v[r][key]
            rows = np.nonzero(dif.any(1))[0]
            print(r, key, name, "ndiff", int(dif.sum()), "rows", rows[:10], "maxabs", float(np.abs(u[r][key] - v[r][key]).max()))
