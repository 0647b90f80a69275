#!/bin/bash
# compute-sanitizer tiers over tools/sanitize_cases.py; summary in
# gpurun_out/sanitize_summary.log, full logs in gpurun_out/sanitize_<tool>_<case>.log.
#   TOOLS="memcheck racecheck synccheck initcheck" CASES="bb1 ragged ..." bash tools/sanitize.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS=$(command -v compute-sanitizer || echo /usr/local/cuda/bin/compute-sanitizer)
TOOLS=${TOOLS:-memcheck racecheck synccheck initcheck}
CASES=${CASES:-bb1 ragged packed lrmsd fa3 long dl cluster serial segment paper precise}
: > gpurun_out/sanitize_summary.log
for t in $TOOLS; do
  for c in $CASES; do
    extra=""
    [ "$t" = "racecheck" ] && extra="--racecheck-report all"
    [ "$c" = "serial" ] && export TPL_PACKED=0
    timeout 900 $CS --tool $t $extra --error-exitcode 99 --print-limit 20 python tools/sanitize_cases.py $c \
      > gpurun_out/sanitize_${t}_${c}.log 2>&1
    rc=$?
    unset TPL_PACKED
    errs=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize_${t}_${c}.log | tail -1)
    echo "$t $c rc=$rc $errs" | tee -a gpurun_out/sanitize_summary.log
  done
done
