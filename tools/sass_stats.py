#!/usr/bin/env python3
"""Per-kernel SASS statistics of libtpl.so (static instruction mix; evidence
that the kernels use TMA bulk copies (UBLKCP) and no local-memory spills).

    python tools/sass_stats.py [filter-substring]
"""
import collections
import re
import subprocess
import sys

LIB = "paper_1812_01108_b200/libtpl.so"


def main():
    flt = sys.argv[1] if len(sys.argv) > 1 else ""
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if flt not in name:
            continue
        ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", f)
        c = collections.Counter(ops)
        total = sum(c.values())
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        top = ", ".join(f"{k} {v}" for k, v in c.most_common(10))
        print(f"{dem}\n   {total} instr | {top}\n   UBLKCP={c.get('UBLKCP', 0)} LDL={c.get('LDL', 0)} "
              f"STL={c.get('STL', 0)} SHFL={c.get('SHFL', 0)} MUFU={c.get('MUFU', 0)}")


if __name__ == "__main__":
    main()
