B="python bench.py --no-cpu-baseline --no-e2e"
timeout 300 $B --mode ag --compressor layerwise > gpurun_out/r2y_bench_layerwise.json 2>/dev/null
timeout 300 python tools/diag_segments.py > gpurun_out/r2y_segments.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2y_launches_layerwise.csv \
  $B --mode ag --compressor layerwise --steps 2 --warmup 3 > gpurun_out/r2y_ncu_lw.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_compressors.py tests/test_gpu_parity.py -x -q > gpurun_out/r2y_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2y_pytest.log
timeout 300 python bench.py > gpurun_out/r2y_bench_n1.json 2> gpurun_out/r2y_bench_n1.err
