#!/usr/bin/env python3
"""Summarise ncu outputs from gpurun_out/ into profiles/ (tracked evidence).

    python tools/summarize_profiles.py --cfg metric --kernel bb_backward --round r01

Writes profiles/<round>_launches_<cfg>.md (per-kernel launch statistics of the
bench command: count, mean device time, share of the kernel time, DRAM bytes
per launch), profiles/<round>_full_<cfg>_<kernel>.md (key --set full metrics
of the dominant kernel) and profiles/traffic_<model>_<cfg>.json (DRAM bytes per
launch that bench.py reports as roofline.traffic).
"""
import argparse
import csv
import json
import os
import statistics
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    idx = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(lambda: defaultdict(dict))
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) != len(hdr):
            continue
        name = r[idx["Kernel Name"]]
        val = float(r[idx["Metric Value"]].replace(",", ""))
        per[name][r[idx["ID"]]][r[idx["Metric Name"]]] = val
    return per


def short(name):
    return name.split("(")[0].replace("void ", "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="metric")
    ap.add_argument("--kernel", default="bb_backward")
    ap.add_argument("--round", default="r01")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    lp = os.path.join(OUT, f"launches_{a.cfg}.csv")
    per = launches(lp)
    tot = sum(sum(m.get("gpu__time_duration.sum", 0) for m in v.values()) for k, v in per.items() if "tpl::" in k)
    lines = [f"# ncu launch list — bench.py --config {a.cfg} (cold-cache, serialised: compare shares)", "",
             "| kernel | launches | mean ns | share of tpl kernel time | DRAM read B/launch | DRAM write B/launch |",
             "|---|---|---|---|---|---|"]
    traffic = {}
    for k, v in sorted(per.items(), key=lambda kv: -sum(m.get("gpu__time_duration.sum", 0) for m in kv[1].values())):
        if "tpl::" not in k:
            continue
        t = [m["gpu__time_duration.sum"] for m in v.values() if "gpu__time_duration.sum" in m]
        rd = [m.get("dram__bytes_read.sum", 0) for m in v.values()]
        wr = [m.get("dram__bytes_write.sum", 0) for m in v.values()]
        lines.append(f"| `{short(k)}` | {len(t)} | {statistics.mean(t):.0f} | {sum(t) / tot * 100:.1f}% | "
                     f"{statistics.mean(rd):.0f} | {statistics.mean(wr):.0f} |")
        kind = "fwd" if "forward" in k else "bwd" if "backward" in k else None
        if kind:
            traffic[kind] = int(statistics.mean(rd) + statistics.mean(wr))
    with open(os.path.join(PROF, f"{a.round}_launches_{a.cfg}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    rep = os.path.join(OUT, f"full_{a.cfg}_{a.kernel}.ncu-rep")
    if os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(raw.splitlines()))
        hdr = rr[0]
        idx = {h: i for i, h in enumerate(hdr)}
        keep = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
                "Executed Ipc Active", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
                "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size",
                "Dynamic Shared Memory Per Block", "L2 Hit Rate", "L1/TEX Hit Rate", "Avg. Active Threads Per Warp"]
        seen, out = set(), [f"# ncu --set full — `{a.kernel}` in bench.py --config {a.cfg}", "",
                            "| metric | value |", "|---|---|"]
        kname = ""
        for r in rr[1:]:
            m = r[idx["Metric Name"]]
            kname = r[idx["Kernel Name"]]
            if m in keep and m not in seen:
                seen.add(m)
                out.append(f"| {m} | {r[idx['Metric Value']]} {r[idx['Metric Unit']]} |")
        raw2 = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        r2 = list(csv.reader(raw2.splitlines()))
        if len(r2) >= 3:
            h2, units, vals = r2[0], r2[1], r2[2]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
            d = {h: (v, u) for h, u, v in zip(h2, units, vals)}

            def nbytes(key):
                v, u = d.get(key, ("0", "byte"))
                return float(v.replace(",", "") or 0) * scale.get(u.strip(), 1)

            rd = nbytes("dram__bytes_read.sum")
            wr = nbytes("dram__bytes_write.sum")
            out.append(f"| dram__bytes_read.sum | {rd:.0f} |")
            out.append(f"| dram__bytes_write.sum | {wr:.0f} |")
            kind = "bwd" if "backward" in a.kernel else "fwd"
            traffic[kind] = int(rd + wr)
        out.insert(1, f"Kernel: `{kname[:140]}`")
        with open(os.path.join(PROF, f"{a.round}_full_{a.cfg}_{a.kernel}.md"), "w") as f:
            f.write("\n".join(out) + "\n")
    model = "backbone" if a.kernel.startswith("bb") else "fullatom"
    with open(os.path.join(PROF, f"traffic_{model}_{a.cfg}.json"), "w") as f:
        json.dump({**traffic, "source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum per launch ({a.round})"},
                  f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
