timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_ef|k_select_x|k_agg_update" --launch-skip 9 --launch-count 3 \
  -o gpurun_out/r2z_ncu_full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2z_ncu_full.log 2>&1
