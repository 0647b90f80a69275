#!/bin/bash
# Full-atom coordinate backward: GPU parity + timings (TPL_FAX shapes) on configs 3 and 5.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullatom.py -x -q -s > gpurun_out/pytest_fa.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_fa.log
grep -E "config3|passed|failed|Error|error" gpurun_out/pytest_fa.log | tail -12
for c in 3 5; do
  for sh in ${SHAPES:-128x1}; do
    echo "config $c TPL_FAX=$sh"
    TPL_FAX=$sh timeout 600 python bench.py --no-cpu-baseline --no-e2e --config $c --steps ${STEPS:-20} --repeats 3 > gpurun_out/fax_${c}_$sh.log 2>&1
    python - gpurun_out/fax_${c}_$sh.log <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d = json.loads(ln); r = d["roofline"]
        print("  value %.3e res/s  step %.4f ms  fwd %.4f ms  bwd %.4f ms (%.0f GB/s)" % (d["value"], d["ms_per_step"], r["fwd"]["ms"], r["bwd"]["ms"], r["bwd"]["GB/s"]))
PY
  done
done
