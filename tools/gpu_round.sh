#!/bin/bash
# One gpurun call: environment facts, GPU tests, smoke, bench.  Logs under gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{ nvidia-smi; nproc; lscpu | head -20; python -c "import torch;p=torch.cuda.get_device_properties(0);print(p, p.L2_cache_size)"; } > gpurun_out/env.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -s ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/smoke.log; tail -c 3000 gpurun_out/bench.log
