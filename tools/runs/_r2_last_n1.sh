timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2last_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2last_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2last_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2last_smoke.log
timeout 300 python bench.py > gpurun_out/r2last_bench_n1.json 2> gpurun_out/r2last_bench_n1.err
