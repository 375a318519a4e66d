"""Top SASS instructions by warp-stall samples from an ncu report (source page).
usage: python profiles/hot_sass.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
data = [dict(zip(h, r)) for r in rows[hdr + 1:] if len(r) == len(h) and r[0] != "Address" and r[2].isdigit()]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print(f"total samples {tot}, instructions {len(data)}")
seen = set()
for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0)):
    if d["Address"] in seen: continue
    seen.add(d["Address"])
    if len(seen) > n: break
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{s:7d} {100*s/max(tot,1):5.1f}%  {d['Address'][-5:]}  {d['Source'].strip()[:90]}")
