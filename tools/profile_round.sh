#!/bin/bash
# One gpurun call producing the round's evidence: a full bench line (cpu_baseline,
# e2e, clocks), the ncu launch list of the same bench command, and one
# `ncu --set full` capture of the dominant kernel.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-metric}
KERN=${KERN:-bb_backward}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{ nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem --format=csv; nproc; lscpu | grep 'Model name'; } > gpurun_out/env.log 2>&1
python bench.py --config $CFG > gpurun_out/bench_full_$CFG.log 2>&1
echo "bench exit $?"
SMALL="python bench.py --config $CFG --steps 4 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e"
$SMALL > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 \
    --csv --log-file gpurun_out/launches_$CFG.csv $SMALL > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?"
$SMALL > gpurun_out/bench_small2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KERN -s 4 -c 1 \
    -o gpurun_out/full_${CFG}_$KERN -f $SMALL > gpurun_out/ncu_full.log 2>&1
echo "full exit $?"
tail -c 600 gpurun_out/bench_full_$CFG.log
