export OMP_NUM_THREADS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2_pytest5.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest5.log
timeout 300 python tools/diag_select.py 138000000 0.01 > gpurun_out/r2_sel5_c3.txt 2>&1
timeout 300 python tools/diag_select.py 355000000 0.1 > gpurun_out/r2_sel5_c4_cr01.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench5.json 2> gpurun_out/r2_bench5.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_select_x --launch-skip 2 --launch-count 1 -o gpurun_out/r2_ncu_sx_c3 -f python tools/diag_select.py 138000000 0.01 > gpurun_out/r2_ncu_sx_c3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_select_x --launch-skip 2 --launch-count 1 -o gpurun_out/r2_ncu_sx_c4 -f python tools/diag_select.py 355000000 0.1 > gpurun_out/r2_ncu_sx_c4.log 2>&1
