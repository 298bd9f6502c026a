# one-GPU run: parity suite, bench with the in-place aggregate vs the dense
# rewrite, the CR crossover of the two, ncu launch list of the step
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2g_gpu.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2g_bench_n1.json 2> gpurun_out/r2g_bench_n1.err
FC_INCR_DIV=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2g_bench_n1_dense.json 2> gpurun_out/r2g_bench_n1_dense.err
for cr in 0.003 0.02 0.03 0.05 0.1; do
  FC_INCR_DIV=1 timeout 300 python bench.py --cr $cr --no-cpu-baseline --no-e2e > gpurun_out/r2g_cr${cr}_inplace.json 2>/dev/null
  FC_INCR_DIV=0 timeout 300 python bench.py --cr $cr --no-cpu-baseline --no-e2e > gpurun_out/r2g_cr${cr}_dense.json 2>/dev/null
done
timeout 600 python bench.py --mode var --no-cpu-baseline --no-e2e > gpurun_out/r2g_bench_n1_var.json 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2g_pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2g_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2g_ncu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2g_smoke.log
