# Same-box A/B of two builds of libtpl.so (TPL_LIB): build/libtpl_old.so vs the in-tree one.
OLD=paper_1812_01108_b200/build/libtpl_old.so
for r in 1 2; do
  for cfg in ${CONFIGS:-2 metric}; do
    for v in old new; do
      if [ $v = old ]; then export TPL_LIB=$OLD; else unset TPL_LIB; fi
      timeout 200 python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.log 2>&1
      echo "run=$r cfg=$cfg $v $(grep -o '"fwd": {"ms": [0-9.e-]*' gpurun_out/ab_$v.log) $(grep -o '"bwd": {"ms": [0-9.e-]*' gpurun_out/ab_$v.log) $(grep -o '"ms_per_step": [0-9.e-]*' gpurun_out/ab_$v.log)" >> gpurun_out/ab_summary.log
    done
  done
done
