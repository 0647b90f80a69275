#!/bin/bash
# Round-end evidence: metric bench line (cpu_baseline, e2e, clocks) + launch list +
# --set full of the forward; then the other configs' bench lines.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
CFG=metric KERN=bb_forward_kernel bash tools/profile_round.sh
for c in ${CONFIGS:-2 3 4 5 lrmsd long}; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_full_$c.log 2>&1; echo "bench $c exit $?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"; tail -c 400 gpurun_out/bench_ref.log
