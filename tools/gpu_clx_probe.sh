#!/bin/bash
# Cluster-split coordinate backward (TPL_BBXC=NTxRPTxCL): parity, then times.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 200 python -m pytest tests/test_gpu_backbone.py -x -q -k "cluster_split or gate or config2" 2>&1 | tail -2
for s in 128x3x2 256x3x2 128x5x2; do
  echo "== $s"
  TPL_BBXC=$s timeout 200 python -m pytest tests/test_gpu_backbone.py -x -q -k "from_coords" 2>&1 | tail -2
  for BL in "64 700" "148 700" "256 700" "128 1000" "256 1000" "32 300"; do
    set -- $BL
    TPL_BBXC=$s timeout 60 python tools/step_timing.py --B $1 --L $2 --xyz | sed "s/^/$s /; s/ sets=[0-9]*//; s/(sum.*//"
  done
done
for BL in "64 700" "148 700" "256 700" "128 1000" "256 1000" "32 300"; do
  set -- $BL
  TPL_BBXC=0 timeout 60 python tools/step_timing.py --B $1 --L $2 --xyz | sed "s/^/default /; s/ sets=[0-9]*//; s/(sum.*//"
done
