B="python bench.py --no-cpu-baseline --no-e2e"
timeout 1200 python -m pytest tests/test_gpu_compressors.py -x -q > gpurun_out/r2m_pytest_comp.log 2>&1; echo rc=$? >> gpurun_out/r2m_pytest_comp.log
timeout 300 $B --mode ag --compressor layerwise > gpurun_out/r2m_bench_layerwise.json 2> gpurun_out/r2m_bench_layerwise.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2m_launches_layerwise.csv \
  $B --mode ag --compressor layerwise --steps 2 --warmup 3 > gpurun_out/r2m_ncu_lw.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2m_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2m_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2m_smoke.log
