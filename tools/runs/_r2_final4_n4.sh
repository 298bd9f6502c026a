# final multi-GPU validation of the round's last code: tests, bench lines,
# two-stage broadcast A/B at N=4, timelines
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r2u_pytest_mg.log 2>&1; echo rc=$? >> gpurun_out/r2u_pytest_mg.log
for N in 2 4; do
  for cfg in "star ring" "star tree" "var ring" "ag ring"; do
    set -- $cfg
    timeout 300 $TR --nproc-per-node $N --master-port 2995$N bench.py --gpus $N --mode $1 --algo $2 --no-e2e \
      > gpurun_out/r2u_bench_n${N}_$1_$2.json 2> gpurun_out/r2u_bench_n${N}_$1_$2.err
  done
done
for a in ring tree; do
  FC_TWO_STAGE_MIN=3 timeout 300 $TR --nproc-per-node 4 --master-port 29964 bench.py --gpus 4 --algo $a --no-e2e \
    > gpurun_out/r2u_bench_n4_star_${a}_twostage.json 2> gpurun_out/r2u_bench_n4_star_${a}_twostage.err
  timeout 300 $TR --nproc-per-node 4 --master-port 29814 tools/diag_mp_timeline.py star $a > gpurun_out/r2u_tl_n4_$a.txt 2>&1
done
timeout 300 $TR --nproc-per-node 4 --master-port 29971 bench.py --gpus 4 --steps 20 --warmup 5 \
  > gpurun_out/r2u_bench_n4_star_e2e.json 2> gpurun_out/r2u_bench_n4_star_e2e.err
