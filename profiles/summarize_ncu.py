"""Summarise ncu output for profiles/ (committed evidence).

  python profiles/summarize_ncu.py launches LAUNCHES.csv STEPS OUT.md
      per-kernel share of the device time from an `ncu --metrics gpu__time_duration.sum`
      launch list (cold-cache, serialised; compare SHARES, not absolutes)
  python profiles/summarize_ncu.py full REPORT.ncu-rep OUT.json OUT.md [CONFIG_JSON]
      per-launch duration, DRAM bytes, tensor-pipe %, issue % and top stall reasons of a
      `--set full` capture; OUT.json holds the GEMM DRAM traffic per step read by bench.py,
      with the captured configuration (bench.py attaches the traffic only to that config)
"""
import collections
import csv
import io
import json
import subprocess
import sys

GEMM_NAMES = ["expert_fc1", "expert_fc2", "expert_dfc2", "expert_dfc1", "expert_dw2", "expert_dw1"]


def launches(path, steps, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v):.1f} | {sum(v) / tot:.1%} |")
    open(out, "w").write(f"# ncu launch list ({path}), {steps} profiled steps\n\n"
                         "Cold-cache serialised durations (`gpu__time_duration.sum`, "
                         "`--clock-control none`): compare shares, not absolutes.\n\n"
                         + "\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out_json, out_md, config=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    recs = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        st = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(d[k])
              for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")
              and d[k] not in ("", "n/a")}
        top = sorted(((v, k) for k, v in st.items() if k not in ("selected",)), reverse=True)[:3]
        recs.append(dict(
            kernel=d["Kernel Name"].split("(")[0].replace("void ", ""),
            us=float(d["gpu__time_duration.sum"]),
            dram_read_MB=float(d["dram__bytes_read.sum"]), dram_write_MB=float(d["dram__bytes_write.sum"]),
            tensor_pct=float(d.get("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed") or 0),
            issue_pct=float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
            dram_pct=float(d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed") or 0),
            regs=int(float(d["launch__registers_per_thread"])), grid=int(float(d["launch__grid_size"])),
            top_stalls=[f"{k} {v:.2f}" for v, k in top]))
    gemms = [r for r in recs if "tc_gemm" in r["kernel"]]
    summary = {"source": rep, "launches": recs}
    if config:
        summary["config"] = json.loads(config)
    if len(gemms) == 6:
        for name, r in zip(GEMM_NAMES, gemms):
            r["op"] = name
        summary["dram_bytes_per_step"] = sum((r["dram_read_MB"] + r["dram_write_MB"]) * 1e6 for r in gemms)
        summary["note"] = ("dram bytes summed over the 6 tcgen05 GEMM launches of one fwd+bwd step "
                           "(ncu --set full, MB = 1e6 B)")
    json.dump(summary, open(out_json, "w"), indent=1)
    lines = ["| launch | op | us | DRAM rd MB | DRAM wr MB | DRAM % | tensor % | issue % | regs | grid | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in recs:
        lines.append(f"| `{r['kernel'][:40]}` | {r.get('op', '')} | {r['us']:.1f} | {r['dram_read_MB']:.1f} | "
                     f"{r['dram_write_MB']:.1f} | {r['dram_pct']:.1f} | {r['tensor_pct']:.1f} | {r['issue_pct']:.1f} | "
                     f"{r['regs']} | {r['grid']} | {', '.join(r['top_stalls'])} |")
    open(out_md, "w").write(f"# ncu --set full summary ({rep})\n\n" + "\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5] if len(sys.argv) > 5 else None)
