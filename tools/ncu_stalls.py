#!/usr/bin/env python3
"""Aggregate warp-stall samples of an ncu source-page CSV (per kernel):
    ncu -i rep --page source --csv --print-source=sass > src.csv; python tools/ncu_stalls.py src.csv"""
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and r:
            cur["rows"].append(r)
    for b in blocks:
        hdr = b["hdr"]
        idx = {h: i for i, h in enumerate(hdr)}
        cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        tot = {c: sum(int(r[idx[c]] or 0) for r in b["rows"]) for c in cols}
        s = sum(tot.values())
        n_sass = len(b["rows"])
        print(f"{b['name'][:90]}\n  SASS instructions {n_sass}, samples {s}")
        for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
            print(f"    {c:28s} {v:6d} {100.0 * v / max(s, 1):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])


def top(path, kernel_substr, n=25):
    rows = list(csv.reader(open(path)))
    cur, hdr = None, None
    out = []
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = r[1]
        elif r and r[0] == "Address":
            hdr = r
        elif cur and kernel_substr in cur and r and hdr:
            out.append(r)
    idx = {h: i for i, h in enumerate(hdr)}
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    S = "Warp Stall Sampling (All Samples)"
    for i, r in enumerate(out):
        r.append(i)
    for r in sorted(out, key=lambda r: -int(r[idx[S]] or 0))[:n]:
        st = sorted(((int(r[idx[c]] or 0), c[6:]) for c in cols), reverse=True)[:2]
        print(f"{r[idx[S]]:>5} #{r[-1]:<5} {r[idx['Source']].strip()[:60]:60s} {st}")
