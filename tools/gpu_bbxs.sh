#!/bin/bash
# Coordinate backward for more chains than SMs: the default single-buffered 128 x 3
# vs the double-buffered 128 x 3 (TPL_BBX=128x3 forces the bbx_shape path).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for x in single double; do
  if [ $x = double ]; then export TPL_BBX=128x3; else unset TPL_BBX; fi
  for BL in "4096 700" "1024 700" "512 1000" "2048 2000"; do set -- $BL
    timeout 120 python tools/step_timing.py --B $1 --L $2 --xyz | sed "s/^/$x /; s/ sets=[0-9]*//; s/(sum.*//"
  done
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --config 4 --steps 50 > gpurun_out/bbxs_$x.json 2>gpurun_out/bbxs_$x.err
  python - gpurun_out/bbxs_$x.json $x <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d = json.loads(ln); r = d["roofline"]
        print("%s config4 step %.4f ms fwd %.4f bwd %.4f" % (sys.argv[2], d["ms_per_step"], r["fwd"]["ms"], r["bwd"]["ms"]))
PY
done
