#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in ${CFGS:-metric 2 3 4}; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --config $c --steps ${STEPS:-50} > gpurun_out/bench_c$c.log 2>&1; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_c*.log")):
    for ln in open(f):
        if ln.startswith("{"):
            d=json.loads(ln); r=d["roofline"]
            print(f, "value %.3e"%d["value"], "ms/step %.4f"%d["ms_per_step"], "fwd %.4f ms %.0f GB/s"%(r["fwd"]["ms"], r["fwd"]["GB/s"]), "bwd %.4f ms %.0f GB/s"%(r["bwd"]["ms"], r["bwd"]["GB/s"]), "step_frac %.3f"%r["step_frac"])
    else:
        print(f, open(f).read()[-800:])
PY
