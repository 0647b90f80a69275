#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
echo "== default"; python tools/latency_sweep.py 2>&1 | tee gpurun_out/sweep_default.log
for nt in ${NTS:-}; do echo "== NT=$nt"; TPL_BB_NT=$nt python tools/latency_sweep.py 2>&1 | tee gpurun_out/sweep$nt.log; done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; tail -c 1500 gpurun_out/bench.log
