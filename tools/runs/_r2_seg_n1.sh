# one-GPU: merged in-place aggregate kernel, layerwise segmented launches --
# bench lines, launch lists, the GPU suite
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/r2k_bench_n1.json 2> gpurun_out/r2k_bench_n1.err
for cr in 0.003 0.015 0.02; do
  FC_INCR_DIV=1 timeout 300 $B --cr $cr > gpurun_out/r2k_cr${cr}_inplace.json 2>/dev/null
  FC_INCR_DIV=0 timeout 300 $B --cr $cr > gpurun_out/r2k_cr${cr}_dense.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2k_launches.csv \
  $B --steps 3 --warmup 3 > gpurun_out/r2k_ncu.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_compressors.py -x -q > gpurun_out/r2k_pytest_comp.log 2>&1; echo rc=$? >> gpurun_out/r2k_pytest_comp.log
timeout 300 $B --mode ag --compressor layerwise > gpurun_out/r2k_bench_layerwise.json 2> gpurun_out/r2k_bench_layerwise.err
timeout 300 $B --mode ag --compressor threshold > gpurun_out/r2k_bench_threshold.json 2> gpurun_out/r2k_bench_threshold.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2k_launches_layerwise.csv \
  $B --mode ag --compressor layerwise --steps 2 --warmup 3 > gpurun_out/r2k_ncu_lw.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2k_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2k_pytest_gpu.log
