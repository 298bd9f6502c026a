export OMP_NUM_THREADS=1
for r in a b; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_l2hint_on_$r.json 2>/dev/null
FC_L2HINT=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_l2hint_off_$r.json 2>/dev/null
done
timeout 300 python tools/diag_select.py 138000000 0.01 > gpurun_out/r2_sel12_c3.txt 2>&1
FC_L2HINT=0 timeout 300 python tools/diag_select.py 138000000 0.01 > gpurun_out/r2_sel12_c3_off.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "trajectory or topk_exact or c1" > gpurun_out/r2_pytest12.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest12.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_prof_bench.json 2> gpurun_out/r2_prof_bench.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_launches.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_ef|k_select_x|k_decode_ar" --launch-skip 9 --launch-count 3 \
  -o gpurun_out/r2_ncu_full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_full.log 2>&1
