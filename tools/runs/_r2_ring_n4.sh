export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for a in ring tree; do
  timeout 300 $TR --nproc-per-node 4 --master-port 29814 tools/diag_mp_timeline.py star $a > gpurun_out/r2r_tl_n4_$a.txt 2>&1
done
for N in 4 2; do
  for cfg in "star ring" "star tree" "var ring"; do
    set -- $cfg
    timeout 300 $TR --nproc-per-node $N --master-port 2995$N bench.py --gpus $N --mode $1 --algo $2 --no-e2e \
      > gpurun_out/r2r_bench_n${N}_$1_$2.json 2> gpurun_out/r2r_bench_n${N}_$1_$2.err
  done
done
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r2r_pytest_mg.log 2>&1; echo rc=$? >> gpurun_out/r2r_pytest_mg.log
