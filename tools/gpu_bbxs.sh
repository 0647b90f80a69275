#!/bin/bash
# Coordinate backward: double-buffered 128 x 3 (default for B > SMs) vs single-buffered (TPL_BBXS=1).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for x in 0 1; do
  if [ $x = 1 ]; then export TPL_BBXS=1; else unset TPL_BBXS; fi
  for BL in "4096 700" "1024 700" "512 1000" "2048 2000" "200 1500"; do set -- $BL
    timeout 120 python tools/step_timing.py --B $1 --L $2 --xyz | sed "s/^/bbxs=$x /; s/ sets=[0-9]*//; s/(sum.*//"
  done
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --config 4 --steps 50 > gpurun_out/bbxs_$x.json 2>gpurun_out/bbxs_$x.err
  python - gpurun_out/bbxs_$x.json $x <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d = json.loads(ln); r = d["roofline"]
        print("bbxs=%s config4 step %.4f ms fwd %.4f bwd %.4f" % (sys.argv[2], d["ms_per_step"], r["fwd"]["ms"], r["bwd"]["ms"]))
PY
done
