#!/bin/bash
# Cluster-split forward (TPL_BBFC=NTxRPTxCL) trials: parity on the ragged-tile
# and metric tests, then the forward/step time at the headline and config 2.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python tools/step_timing.py --B 256 --L 700 --xyz
for s in ${SHAPES:-128x3x2 128x5x2 64x7x2 64x3x4 128x1x8 32x3x8}; do
  echo "== $s"
  TPL_BBFC=$s timeout 200 python -m pytest tests/test_gpu_backbone.py -x -q -k "ragged_tiles or config1 or config2 or metric or gate or determinism" 2>&1 | tail -2
  TPL_BBFC=$s timeout 60 python tools/step_timing.py --B 256 --L 700 --xyz
  TPL_BBFC=$s timeout 60 python tools/step_timing.py --B 64 --L 700 --xyz
  TPL_BBFC=$s timeout 60 python tools/step_timing.py --B 512 --L 700 --xyz
done
