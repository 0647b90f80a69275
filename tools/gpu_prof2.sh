#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for CFG in metric 4; do
python tools/prof_driver.py --config $CFG --iters 4 --sets 2 > gpurun_out/prof_plain_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"bb_" -s 2 -c 2 \
    -o gpurun_out/prof_$CFG -f python tools/prof_driver.py --config $CFG --iters 4 --sets 2 > gpurun_out/ncu_full_$CFG.log 2>&1
echo "$CFG exit $?"
done
