export OMP_NUM_THREADS=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compressors.py tests/test_gpu_async.py -x -q > gpurun_out/r2_pytest4.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest4.log
timeout 300 python tools/diag_select.py 138000000 0.01 > gpurun_out/r2_sel4_c3.txt 2>&1
timeout 300 python tools/diag_select.py 355000000 0.1 > gpurun_out/r2_sel4_c4_cr01.txt 2>&1
timeout 300 python tools/diag_step.py > gpurun_out/r2_diag_step4.jsonl 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench4.json 2> gpurun_out/r2_bench4.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --mode ag > gpurun_out/r2_bench4_ag.json 2> gpurun_out/r2_bench4_ag.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_pytest4_full.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest4_full.log
