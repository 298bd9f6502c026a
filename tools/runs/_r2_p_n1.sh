timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2p_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2p_pytest_gpu.log
timeout 300 python bench.py > gpurun_out/r2p_bench_n1.json 2> gpurun_out/r2p_bench_n1.err
