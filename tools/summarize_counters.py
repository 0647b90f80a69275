#!/usr/bin/env python3
"""Summarise tools/counters.sh CSVs (ncu --metrics ... --csv) into a markdown table:
    python tools/summarize_counters.py gpurun_out/counters_*.csv > profiles/r02_counters.md"""
import csv
import os
import re
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "wait", "no_instruction", "math_pipe_throttle",
          "mio_throttle", "lg_throttle", "branch_resolving", "dispatch_stall"]


def algo_bytes(cfg, kname):
    """Algorithmic bytes per launch."""
    c = synth.CONFIGS[cfg]
    if c["model"] == "backbone":
        _, ln, _ = synth.backbone_inputs(cfg)
        r = int(ln.sum())
        if "lrmsd_kernel" in kname:
            return 60 * r
        if "chain_scale" in kname:
            return 24 * r
        return (48 if "forward" in kname else 60) * r
    ang, rt, ln = synth.fullatom_inputs(cfg)
    table = synth.load_residue_table()
    per = [len(t["atoms"]) for t in table["types"]]
    atoms = sum(per[int(t)] for b in range(rt.shape[0]) for t in rt[b, : int(ln[b])])
    r = int(ln.sum())
    return (33 * r + 12 * atoms) if "forward" in kname else (65 * r + 12 * atoms)


def main(paths):
    print("# Round 2 — ncu counters of the dominant kernels (tools/counters.sh, B200)\n")
    print("One short `bench.py` run per config under `ncu --metrics` (kernels replayed with caches flushed, clocks "
          "unlocked): times are serialised cold-cache per launch, so compare the counters, not the absolute times. "
          "fp32 flop = 2 FFMA + FADD + FMUL + 4 FFMA2 + 2 FADD2 + 2 FMUL2 (thread instructions). FMA pipe % = "
          "`sm__pipe_fma_cycles_active` of peak; XU = MUFU/conversion warp instructions; stalls = the top three "
          "`smsp__average_warps_issue_stalled_*_per_issue_active` ratios (warps stalled per issued instruction).\n")
    print("| config | kernel | launches | ncu us/launch | FMA pipe % | ALU pipe % | fp32 TFLOP/s | XU inst/launch | "
          "warps active % | issue active % | top stalls | DRAM MB/launch | algorithmic MB | DRAM / algorithmic |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        cfg = re.search(r"counters_(.+)\.csv", p).group(1)
        key = synth.register_custom(cfg) if ":" in cfg else (cfg if cfg in synth.CONFIGS else int(cfg))
        rows = [r for r in csv.reader(open(p)) if len(r) > 10]
        hdr = rows[0]
        idx = {h: i for i, h in enumerate(hdr)}
        per = defaultdict(lambda: defaultdict(list))
        for r in rows[1:]:
            k = re.sub(r"\(.*", "", r[idx["Kernel Name"]]).replace("tpl::", "")
            per[k][r[idx["Metric Name"]]].append(float(r[idx["Metric Value"]].replace(",", "")))
        for k, m in sorted(per.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
            n = len(m["gpu__time_duration.sum"])
            avg = lambda name: sum(m[name]) / max(len(m[name]), 1)  # noqa: E731
            t_ns = avg("gpu__time_duration.sum")
            flops = (2 * avg("sm__sass_thread_inst_executed_op_ffma_pred_on.sum") + avg(
                "sm__sass_thread_inst_executed_op_fadd_pred_on.sum") + avg(
                "sm__sass_thread_inst_executed_op_fmul_pred_on.sum") + 4 * avg(
                "sm__sass_thread_inst_executed_op_ffma2_pred_on.sum") + 2 * avg(
                "sm__sass_thread_inst_executed_op_fadd2_pred_on.sum") + 2 * avg(
                "sm__sass_thread_inst_executed_op_fmul2_pred_on.sum"))
            st = sorted(((s, avg(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio")) for s in STALLS),
                        key=lambda kv: -kv[1])[:3]
            dram = avg("dram__bytes_read.sum") + avg("dram__bytes_write.sum")
            ab = algo_bytes(key, k)
            print(f"| {cfg} | `{k}` | {n} | {t_ns / 1e3:.2f} | {avg('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f} "
                  f"| {avg('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | {flops / t_ns / 1e3:.2f} "
                  f"| {avg('sm__inst_executed_pipe_xu.sum'):.0f} | {avg('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} "
                  f"| {avg('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
                  + ", ".join(f"{s} {v:.2f}" for s, v in st)
                  + f" | {dram / 1e6:.2f} | {ab / 1e6:.2f} | {dram / ab:.2f} |")


if __name__ == "__main__":
    main(sys.argv[1:])
