#!/bin/bash
# Full-atom forward variants (TPL_FAF=NTxTSxMINB) on configs 3 and 5.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for sh in ${SHAPES:-256x1x2}; do
  TPL_FAF=$sh timeout 300 python -m pytest tests/test_gpu_fullatom.py -x -q -k "config3 and from_coords" > gpurun_out/faf_pytest_$sh.log 2>&1 || echo "PARITY FAIL $sh"
  for c in 3 5; do
    TPL_FAF=$sh timeout 600 python bench.py --no-cpu-baseline --no-e2e --config $c --steps ${STEPS:-20} --repeats 3 > gpurun_out/faf_${c}_$sh.log 2>&1
    python - gpurun_out/faf_${c}_$sh.log $c $sh <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d = json.loads(ln); r = d["roofline"]
        print("config %s %-10s value %.3e res/s  step %.4f ms  fwd %.4f ms  bwd %.4f ms" % (sys.argv[2], sys.argv[3], d["value"], d["ms_per_step"], r["fwd"]["ms"], r["bwd"]["ms"]))
PY
  done
done
