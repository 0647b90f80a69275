#!/bin/bash
# Full-atom forward shape trials on config 5 (TPL_FAF=NTxTSxMINB).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for f in default 128x0x4 128x1x6 128x1x4 256x0x3 256x0x2; do
  if [ $f = default ]; then unset TPL_FAF; else export TPL_FAF=$f; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --config 5 --steps 30 > gpurun_out/faf5.json 2>/dev/null
  python - gpurun_out/faf5.json $f <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d = json.loads(ln); r = d["roofline"]
        print("%-9s config5 step %.4f ms fwd %.4f bwd %.4f" % (sys.argv[2], d["ms_per_step"], r["fwd"]["ms"], r["bwd"]["ms"]))
PY
done
