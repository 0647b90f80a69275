#!/usr/bin/env python3
"""Warp-stall samples of an ncu report aggregated per CUDA source line (needs
-lineinfo and --import-source on):  python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, fname, lines = None, "", []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[0] and r[2] == "-":
            lines.append((fname, r))
    idx = {h: i for i, h in enumerate(hdr)}
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    samp = idx["Warp Stall Sampling (All Samples)"]
    tot = sum(int(r[samp] or 0) for _, r in lines)
    print(f"{rep}: {tot} samples")
    agg = {}
    for f, r in lines:
        s = sum(int(r[idx[c]] or 0) for c in cols)
        agg.setdefault("total", {}).update()
        for c in cols:
            agg.setdefault(c, 0)
            agg[c] += int(r[idx[c]] or 0)
    print("  totals:", sorted(((c[6:], v) for c, v in agg.items() if c != "total"), key=lambda kv: -kv[1])[:8])
    lines.sort(key=lambda fr: -int(fr[1][samp] or 0))
    for f, r in lines[:top]:
        s = int(r[samp] or 0)
        if not s:
            break
        st = sorted(((c[6:], int(r[idx[c]] or 0)) for c in cols), key=lambda kv: -kv[1])[:3]
        print(f"{100.0 * s / tot:5.1f}% {f}:{r[0]:<5} {r[1].strip()[:64]:64s} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
