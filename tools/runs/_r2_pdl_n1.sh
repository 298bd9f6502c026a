for r in a b c; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2pdl_bench_$r.json 2>/dev/null
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2pdl_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2pdl_pytest.log
