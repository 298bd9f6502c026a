export OMP_NUM_THREADS=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compressors.py tests/test_gpu_async.py tests/test_gpu_moo.py tests/test_cpp_facade.py -x -q > gpurun_out/r2_pytest11.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest11.log
FC_DECODE=direct timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "trajectory or c1_full or owed" > gpurun_out/r2_pytest11_direct.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest11_direct.log
timeout 300 python tools/diag_select.py 138000000 0.01 > gpurun_out/r2_sel11_c3.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench11_n1.json 2> gpurun_out/r2_bench11_n1.err
FC_DECODE=direct timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench11_n1_direct.json 2> gpurun_out/r2_bench11_n1_direct.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench11_n1_b.json 2> gpurun_out/r2_bench11_n1_b.err
FC_DECODE=direct timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench11_n1_direct_b.json 2> gpurun_out/r2_bench11_n1_direct_b.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_pytest11_full.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest11_full.log
bash tools/sanitize_one.sh memcheck
