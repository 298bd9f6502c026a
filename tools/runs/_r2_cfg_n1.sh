for cfg in C1 C2 C4 C5 C3-thr C3-tree; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2cfg_$cfg.json 2> gpurun_out/r2cfg_$cfg.err
done
