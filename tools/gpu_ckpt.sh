#!/bin/bash
# Checkpointed backbone pair: GPU parity + per-launch timings vs the plain pair.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_backbone.py -x -q -s > gpurun_out/pytest_bb.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_bb.log
tail -3 gpurun_out/pytest_bb.log
for BL in "256 700" "1 700" "4096 700" "64 2000"; do
  set -- $BL
  timeout 120 python tools/step_timing.py --B $1 --L $2
  timeout 120 python tools/step_timing.py --B $1 --L $2 --ckpt
done
