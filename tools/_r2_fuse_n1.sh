timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2s_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2s_pytest_gpu.log
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 300 python bench.py > gpurun_out/r2s_bench_n1.json 2> gpurun_out/r2s_bench_n1.err
timeout 300 $B --mode var > gpurun_out/r2s_bench_n1_var.json 2>/dev/null
for cr in 0.003 0.0125; do
  timeout 300 $B --cr $cr > gpurun_out/r2s_cr${cr}_inplace.json 2>/dev/null
  FC_INCR_DIV=0 timeout 300 $B --cr $cr > gpurun_out/r2s_cr${cr}_dense.json 2>/dev/null
done
timeout 300 python tools/diag_select.py > gpurun_out/r2s_sel.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2s_launches.csv \
  $B --steps 3 --warmup 3 > gpurun_out/r2s_ncu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2s_smoke.log
