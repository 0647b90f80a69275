#!/bin/bash
# Full GPU test suite, smoke, and bench lines for the BASELINE configs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
for c in ${CONFIGS:-metric 2 3 4 5 lrmsd long}; do
  timeout 600 python bench.py --no-cpu-baseline --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python - gpurun_out/bench_$c.json $c <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d = json.loads(ln); r = d["roofline"]
        print("%-7s value %.3e  step %.4f ms  fwd %.4f  bwd %.4f  frac %.3f  e2e %.3e  clk %s %s" % (sys.argv[2], d["value"], d["ms_per_step"], r["fwd"]["ms"], r["bwd"]["ms"], r["frac"], d["e2e"]["value"], d["clocks"].get("sm_mhz"), d["clocks"].get("reasons")))
PY
done
