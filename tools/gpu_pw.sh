set -x
export TPL_BBX_PW=1
timeout 400 python -m pytest tests/test_gpu_backbone.py tests/test_gpu_fuzz.py tests/test_gpu_lrmsd.py -q -x > gpurun_out/pw_tests.log 2>&1; echo rc=$? >> gpurun_out/pw_tests.log
for pw in 0 1 0 1; do
  for cfg in metric 4; do
    TPL_BBX_PW=$pw timeout 200 python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/pw_bench_${pw}_${cfg}.log 2>&1
    echo "pw=$pw cfg=$cfg $(grep -o '"bwd": {"ms": [0-9.e-]*' gpurun_out/pw_bench_${pw}_${cfg}.log) $(grep -o '"ms_per_step": [0-9.e-]*' gpurun_out/pw_bench_${pw}_${cfg}.log)" >> gpurun_out/pw_summary.log
  done
done
