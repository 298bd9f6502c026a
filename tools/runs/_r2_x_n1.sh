B="python bench.py --no-cpu-baseline --no-e2e"
timeout 300 python tools/diag_segments.py > gpurun_out/r2x_segments.txt 2>&1
timeout 300 $B --mode ag --compressor layerwise > gpurun_out/r2x_bench_layerwise.json 2>/dev/null
timeout 600 python tools/diag_select.py 355000000 0.1 > gpurun_out/r2x_sel_c4_cr01.txt 2>&1
timeout 300 python bench.py > gpurun_out/r2x_bench_n1.json 2> gpurun_out/r2x_bench_n1.err
timeout 300 $B --mode ag --compressor threshold > gpurun_out/r2x_bench_threshold.json 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2x_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2x_pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2x_launches_layerwise.csv \
  $B --mode ag --compressor layerwise --steps 2 --warmup 3 > gpurun_out/r2x_ncu_lw.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2x_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2x_smoke.log
