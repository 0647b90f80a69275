# A/B of the forward's huge-angle redo vote (per-warp __any_sync vs the block-wide
# __syncthreads_or of the previous build): parity, then the metric and config 2/4 lines.
timeout 400 python -m pytest tests/test_gpu_backbone.py tests/test_gpu_fuzz.py tests/test_gpu_lrmsd.py -q -x > gpurun_out/any_tests.log 2>&1; echo rc=$? >> gpurun_out/any_tests.log
for r in 1 2; do
  for cfg in metric 2 4; do
    timeout 200 python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/any_bench_${cfg}.log 2>&1
    echo "run=$r cfg=$cfg $(grep -o '"fwd": {"ms": [0-9.e-]*' gpurun_out/any_bench_${cfg}.log) $(grep -o '"ms_per_step": [0-9.e-]*' gpurun_out/any_bench_${cfg}.log)" >> gpurun_out/any_summary.log
  done
done
