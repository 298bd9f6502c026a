# one-GPU A/B: in-place aggregate write granule (8 / 16 / 32 floats) at three
# CRs, the select's lite pass variant, select phases
B="python bench.py --no-cpu-baseline --no-e2e"
for cr in 0.01 0.003 0.02; do
  for a in 8 16 32; do
    FC_INCR_DIV=1 FC_AGG_ATOM=$a timeout 300 $B --cr $cr > gpurun_out/r2i_cr${cr}_atom$a.json 2>/dev/null
  done
  FC_INCR_DIV=0 timeout 300 $B --cr $cr > gpurun_out/r2i_cr${cr}_dense.json 2>/dev/null
done
FC_SX_LITE=1 timeout 300 $B > gpurun_out/r2i_sxlite.json 2>/dev/null
timeout 300 $B > gpurun_out/r2i_default.json 2>/dev/null
timeout 300 python tools/diag_select.py > gpurun_out/r2i_sel_default.txt 2>&1
FC_SX_LITE=1 timeout 300 python tools/diag_select.py > gpurun_out/r2i_sel_lite.txt 2>&1
FC_INCR_DIV=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2i_launches.csv \
  $B --steps 3 --warmup 3 > gpurun_out/r2i_ncu.log 2>&1
