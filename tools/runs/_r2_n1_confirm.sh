B="python bench.py"
timeout 600 $B > gpurun_out/r2j_bench_n1.json 2> gpurun_out/r2j_bench_n1.err
FC_INCR_DIV=0 timeout 300 $B --no-cpu-baseline --no-e2e > gpurun_out/r2j_bench_n1_dense.json 2>/dev/null
timeout 300 $B --mode var --no-cpu-baseline --no-e2e > gpurun_out/r2j_bench_n1_var.json 2>/dev/null
timeout 300 $B --mode ag --no-cpu-baseline --no-e2e > gpurun_out/r2j_bench_n1_ag.json 2>/dev/null
timeout 300 python tools/diag_select.py > gpurun_out/r2j_sel.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2j_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2j_pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2j_launches.csv \
  $B --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2j_ncu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2j_smoke.log
