export OMP_NUM_THREADS=1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_prof_bench.json 2> gpurun_out/r2_prof_bench.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_launches.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_ef|k_select_x|k_decode_ar" --launch-skip 9 --launch-count 3 \
  -o gpurun_out/r2_ncu_full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_full.log 2>&1
