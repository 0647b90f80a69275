#!/bin/bash
# ncu launch list + one full-set capture per kernel of a config (1 GPU).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-metric}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/prof_driver.py --config $CFG --iters 6 --overhead > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$CFG.csv python tools/prof_driver.py --config $CFG --iters 6 > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"bb_|fa_" -s 4 -c 2 \
    -o gpurun_out/prof_$CFG -f python tools/prof_driver.py --config $CFG --iters 6 > gpurun_out/ncu_full.log 2>&1
echo "exit $?"
cat gpurun_out/prof_plain.log
tail -5 gpurun_out/ncu_full.log
