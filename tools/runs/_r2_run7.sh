export OMP_NUM_THREADS=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compressors.py tests/test_gpu_async.py tests/test_gpu_moo.py tests/test_cpp_facade.py -x -q > gpurun_out/r2_pytest7.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest7.log
timeout 300 python tools/diag_select.py 138000000 0.01 > gpurun_out/r2_sel7_c3.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench7.json 2> gpurun_out/r2_bench7.err
(cd tests/cpp && timeout 300 ./bench_facade 138000000 4) > gpurun_out/r2_bench_facade7.json 2>&1
timeout 300 python tools/diag_step.py > gpurun_out/r2_diag_step7.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_pytest7_full.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest7_full.log
