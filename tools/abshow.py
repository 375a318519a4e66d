"""Print per-op times of the A/B/n bench lines in gpurun_out/ab/ (usage: python tools/abshow.py)."""
import glob
import json
import os

OPS = ["expert_fc1", "expert_fc2", "expert_dfc2", "expert_dfc1", "expert_dw2", "expert_dw1", "gate",
       "permute", "combine", "combine_bwd", "unpermute_gate_bwd", "gate_dwg"]
for f in sorted(glob.glob("gpurun_out/ab/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(os.path.basename(f), "ERR", e)
        continue
    k = d["kernels"]
    print(f"{os.path.basename(f):22s} {d['ms_per_step']:.3f}ms " +
          " ".join(f"{o.replace('expert_', '')}={k[o]['us']:.0f}" for o in OPS if o in k))
