#!/bin/bash
# Newton-Schulz policy sweep (TPL_ORTHO) of the backbone forward: regular-structure
# error (tools/regular_check.py), the random-chain gate, and forward times.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for ns in ${NS_LIST:-1 2 3}; do
  echo "== TPL_ORTHO=$ns"
  TPL_ORTHO=$ns timeout 300 python tools/regular_check.py
  TPL_ORTHO=$ns timeout 300 python -m pytest tests/test_gpu_backbone.py -q -s -k "gate" 2>&1 | grep -E "err|passed|failed"
  for i in 1 2; do TPL_ORTHO=$ns timeout 120 python tools/step_timing.py --B 256 --L 700 --xyz; done
  TPL_ORTHO=$ns timeout 120 python tools/step_timing.py --B 4096 --L 700 --xyz
  TPL_ORTHO=$ns timeout 120 python tools/step_timing.py --B 64 --L 700 --xyz
done
