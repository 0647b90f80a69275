#!/bin/bash
# Cluster-split forward vs the default forward over (B, L) near the switch points.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for BL in ${POINTS:-"256 1000" "512 1000" "64 1500" "16 1500" "256 900" "200 600" "148 600" "8 2500"}; do
  set -- $BL
  echo "== B=$1 L=$2"
  TPL_BBFC=0 timeout 60 python tools/step_timing.py --B $1 --L $2 --xyz | sed 's/^/default  /'
  for s in ${SHAPES:-128x3x2 128x5x2 128x7x2 128x3x4 128x5x4}; do TPL_BBFC=$s timeout 60 python tools/step_timing.py --B $1 --L $2 --xyz | sed "s/^/$s /"; done
done
