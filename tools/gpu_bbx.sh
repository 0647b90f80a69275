#!/bin/bash
# Backbone backward variants: GPU parity + per-launch timings (plain / from-coords, TPL_BBX shapes).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_backbone.py -x -q -s > gpurun_out/pytest_bb.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_bb.log
grep -E "from_coords|single chain|passed|failed|Error|error" gpurun_out/pytest_bb.log | tail -12
# SIZES="256x700 4096x700" (BxL list)
for BL in ${SIZES:-256x700 1x700 4096x700 64x2000}; do
  set -- ${BL/x/ }
  for sh in ${SHAPES:-""}; do TPL_BBF=$sh TPL_BBXD=$sh timeout 120 python tools/step_timing.py --B $1 --L $2 --xyz 2>&1 | tail -1; done
  TPL_DL=0 timeout 120 python tools/step_timing.py --B $1 --L $2 --xyz
  timeout 120 python tools/step_timing.py --B $1 --L $2 --xyz
done
