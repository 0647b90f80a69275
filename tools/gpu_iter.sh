#!/bin/bash
# Iteration run: GPU tests (+ TPL_ORTHO variants on the precision tests) and a bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for ns in 0 2; do
  TPL_ORTHO=$ns timeout 300 python -m pytest tests/test_gpu_backbone.py -q -s -k "config2 or regular" > gpurun_out/ns$ns.log 2>&1; echo "exit $?" >> gpurun_out/ns$ns.log
done
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
for c in 2 4 3; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --config $c --steps 50 > gpurun_out/bench_c$c.log 2>&1; done
grep -E "passed|failed|error|config|helix|strand|extended" gpurun_out/pytest_gpu.log | tail -8
for ns in 0 2; do echo "ns=$ns"; grep -E "config2|helix|strand|extended|passed|failed" gpurun_out/ns$ns.log; done
python - <<'PY'
import json,glob
for f in ["gpurun_out/bench.log"]+sorted(glob.glob("gpurun_out/bench_c*.log")):
    for ln in open(f):
        if ln.startswith("{"):
            d=json.loads(ln); r=d["roofline"]
            print(f, "value %.3e"%d["value"], "ms/step %.4f"%d["ms_per_step"], "fwd %.4f ms %.0f GB/s"%(r["fwd"]["ms"], r["fwd"]["GB/s"]), "bwd %.4f ms %.0f GB/s"%(r["bwd"]["ms"], r["bwd"]["GB/s"]), "step_frac %.3f"%r["step_frac"], "clk", d["clocks"].get("sm_mhz"))
PY
