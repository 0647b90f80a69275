#!/bin/bash
# One parameterised driver for gpurun calls (run from the repo root on the GPU box):
#   tools/gpu.sh tests [pytest -k expr]          GPU test suite (-m gpu)
#   tools/gpu.sh bench CFG...                     full bench lines -> gpurun_out/bench_<cfg>.log
#   tools/gpu.sh ab "ENV_A" "ENV_B" CFG...       same-box A/B of two environments (2 repeats, fwd/bwd/step)
#   tools/gpu.sh launches CFG                     ncu launch list of a short bench run
#   tools/gpu.sh full CFG KERNEL_REGEX            ncu --set full of one launch of a kernel
#   tools/gpu.sh sanitize                         compute-sanitizer tiers (tools/sanitize.sh)
# Several tasks may be chained:  tools/gpu.sh tests -- bench metric 2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
SMALL_ARGS="--steps 4 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e"
field() { grep -o "\"$1\": {\"ms\": [0-9.e-]*" "$2" | grep -o '[0-9.e-]*$'; }
while [ $# -gt 0 ]; do
  task=$1; shift
  args=()
  while [ $# -gt 0 ] && [ "$1" != "--" ]; do args+=("$1"); shift; done
  [ "$1" = "--" ] && shift
  case $task in
    tests)
      timeout 900 python -m pytest tests -m gpu -x -q ${args[0]:+-k "${args[0]}"} > gpurun_out/tests.log 2>&1
      echo "tests exit $?"; tail -3 gpurun_out/tests.log ;;
    bench)
      for c in "${args[@]}"; do
        timeout 600 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo "bench $c exit $?"
        python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
ln = [l for l in open(f"gpurun_out/bench_{c}.log") if l.startswith("{")]
if ln:
    d = json.loads(ln[-1]); r = d["roofline"]
    print(f"  {c}: {d['value']:.4g} res/s step {d['ms_per_step']*1e3:.2f} us fwd {r['fwd']['ms']*1e3:.2f} bwd {r['bwd']['ms']*1e3:.2f} frac {r['frac']} step_frac {r['step_frac']:.3f} parity {d.get('parity')}")
PY
      done ;;
    ab)
      A=${args[0]}; Bv=${args[1]}
      for r in 1 2; do
        for c in "${args[@]:2}"; do
          for v in A B; do
            if [ $v = A ]; then E=$A; else E=$Bv; fi
            env $E timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-parity > gpurun_out/ab_$v.log 2>&1
            echo "run=$r cfg=$c [$E] fwd $(field fwd gpurun_out/ab_$v.log) bwd $(field bwd gpurun_out/ab_$v.log) $(grep -o '"ms_per_step": [0-9.e-]*' gpurun_out/ab_$v.log)"
          done
        done
      done ;;
    launches)
      c=${args[0]}
      python bench.py --config $c $SMALL_ARGS --no-parity > /dev/null 2>&1 && \
      ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -c 400 \
          --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c $SMALL_ARGS --no-parity > gpurun_out/ncu_launch.log 2>&1
      echo "launches $c exit $?" ;;
    full)
      c=${args[0]}; k=${args[1]}
      ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$k -s 4 -c 1 \
          -o gpurun_out/full_${c}_$k -f python bench.py --config $c $SMALL_ARGS --no-parity > gpurun_out/ncu_full_$c.log 2>&1
      echo "full $c $k exit $?" ;;
    sanitize)
      bash tools/sanitize.sh; echo "sanitize exit $?" ;;
    *) echo "unknown task $task"; exit 2 ;;
  esac
done
