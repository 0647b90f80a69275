#!/bin/bash
# Forward chain-per-CTA shape sweep (TPL_BBFS=NTxRPT) on config 4 and 4096 x 700.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for x in default 128x3 128x5 128x7 256x3 256x5; do
  if [ $x = default ]; then unset TPL_BBFS; else export TPL_BBFS=$x; fi
  timeout 120 python tools/step_timing.py --B 4096 --L 700 --xyz | sed "s/^/$x /; s/ sets=[0-9]*//; s/(sum.*//"
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --config 4 --steps 50 > gpurun_out/bbfs.json 2>/dev/null
  python - gpurun_out/bbfs.json $x <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d = json.loads(ln); r = d["roofline"]
        print("%s config4 step %.4f ms fwd %.4f bwd %.4f" % (sys.argv[2], d["ms_per_step"], r["fwd"]["ms"], r["bwd"]["ms"]))
PY
done
