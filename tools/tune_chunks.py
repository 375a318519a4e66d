"""Validate the chunk-count tuner on the GPU.

Runs bench.py on the expert-parallel path (LANCET_FLAG_FORCE_EP on one GPU, or under torchrun
at N > 1) for n = 1, 2, 4, 8 chunks, fits the tuner's cost model on two of them (n = 1, 4),
predicts the step time of all four and reports the prediction error (the paper reports 3.83 %
for its optimizer) and the n the tuner would pick.

    python tools/tune_chunks.py [--flags 512] > gpurun_out/tune.json
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_19429_b200.chunk_tuner import best_n, fit, simulate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--flags", type=int, default=512)
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
lines = {}
for n in (1, 2, 4, 8):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", str(a.steps), "--warmup", "4",
           "--no-e2e", "--no-cpu-baseline", "--chunks", str(n), "--flags", str(a.flags)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines[n] = json.loads(r.stdout.strip().splitlines()[-1])
m = fit({n: lines[n] for n in (1, 4)})
out = {"fit_on": [1, 4], "points": []}
for n in (1, 2, 4, 8):
    p = simulate(m, n)
    meas = lines[n]["ms_per_step"] * 1000.0
    out["points"].append({"n": n, "measured_us": meas, "predicted_us": p["step_us"],
                          "error": (p["step_us"] - meas) / meas,
                          "measured_exposed_us": lines[n]["exposed_a2a_ms"] * 1000.0,
                          "predicted_exposed_us": p["exposed_comm_us"]})
out["tuner_pick"] = best_n(m)[0]
out["measured_best"] = min(lines, key=lambda n: lines[n]["ms_per_step"])
m_all = fit(lines)
out["tuner_pick_fit_all"] = best_n(m_all)[0]
print(json.dumps(out, indent=1))
