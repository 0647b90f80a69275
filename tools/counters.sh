#!/bin/bash
# ncu counters north_star names for the dominant kernels of every config (one short bench
# run each; serialised, caches flushed between replays -- compare shares, not absolutes):
#   CONFIGS="metric 2 3 4 5 lrmsd" bash tools/counters.sh   -> gpurun_out/counters_<cfg>.csv
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
M=$M,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed.sum
M=$M,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum
M=$M,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum
M=$M,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for r in barrier long_scoreboard short_scoreboard wait no_instruction math_pipe_throttle mio_throttle lg_throttle branch_resolving dispatch_stall not_selected selected; do
  M=$M,smsp__average_warps_issue_stalled_${r}_per_issue_active.ratio
done
for c in ${CONFIGS:-metric 2 3 4 5 lrmsd}; do
  timeout 900 ncu --metrics $M --clock-control none --kernel-name-base demangled -k regex:tpl:: -s 12 -c 8 --csv --log-file gpurun_out/counters_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/counters_$c.log 2>&1
  echo "counters $c exit $?"
done
