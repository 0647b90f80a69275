#!/bin/bash
# Full-atom config 3 launch-shape trials (TPL_FAF forward, TPL_FAX coordinate backward).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for f in 256x1x2 512x1x1; do for x in 256x1x0x0 512x1x0x0; do
  TPL_FAF=$f TPL_FAX=$x timeout 300 python -m pytest tests/test_gpu_fullatom.py -x -q -k "config3 and from_coords" > gpurun_out/fa3_$f_$x.log 2>&1 || echo "PARITY FAIL $f $x"
  TPL_FAF=$f TPL_FAX=$x timeout 300 python bench.py --no-cpu-baseline --no-e2e --config 3 --steps 50 --repeats 5 > gpurun_out/fa3b.log 2>&1
  python - gpurun_out/fa3b.log "$f $x" <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d = json.loads(ln); r = d["roofline"]
        print("%-22s step %.4f ms  fwd %.4f  bwd %.4f" % (sys.argv[2], d["ms_per_step"], r["fwd"]["ms"], r["bwd"]["ms"]))
PY
done; done
