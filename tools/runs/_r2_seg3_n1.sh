B="python bench.py --no-cpu-baseline --no-e2e"
timeout 1200 python -m pytest tests/test_gpu_compressors.py tests/test_gpu_moo.py -x -q > gpurun_out/r2n_pytest_comp.log 2>&1; echo rc=$? >> gpurun_out/r2n_pytest_comp.log
timeout 300 $B --mode ag --compressor layerwise > gpurun_out/r2n_bench_layerwise.json 2> gpurun_out/r2n_bench_layerwise.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2n_launches_layerwise.csv \
  $B --mode ag --compressor layerwise --steps 2 --warmup 3 > gpurun_out/r2n_ncu_lw.log 2>&1
timeout 300 $B > gpurun_out/r2n_bench_n1.json 2> gpurun_out/r2n_bench_n1.err
