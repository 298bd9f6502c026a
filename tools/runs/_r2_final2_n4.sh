# 4-GPU run: bench lines (peer memory + NCCL-only), C4 sweep at N=4 and N=2,
# multi-GPU tests, NVLink calibration, NVLink byte counters at N=2
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out/calg
for N in 2 4; do
  for cfg in "star ring" "star tree" "var ring" "ag ring"; do
    set -- $cfg
    timeout 300 $TR --nproc-per-node $N --master-port 2995$N bench.py --gpus $N --mode $1 --algo $2 --no-e2e \
      > gpurun_out/r2h_bench_n${N}_$1_$2.json 2> gpurun_out/r2h_bench_n${N}_$1_$2.err
  done
  FC_INCR_DIV=0 timeout 300 $TR --nproc-per-node $N --master-port 2997$N bench.py --gpus $N --no-e2e \
    > gpurun_out/r2h_bench_n${N}_star_ring_densedecode.json 2> gpurun_out/r2h_bench_n${N}_star_ring_densedecode.err
  for cfg in "star ring" "ag ring"; do
    set -- $cfg
    FC_NO_P2P=1 timeout 300 $TR --nproc-per-node $N --master-port 2996$N bench.py --gpus $N --mode $1 --algo $2 --no-e2e \
      > gpurun_out/r2h_bench_n${N}_$1_$2_nccl.json 2> gpurun_out/r2h_bench_n${N}_$1_$2_nccl.err
  done
done
timeout 300 $TR --nproc-per-node 4 --master-port 29971 bench.py --gpus 4 --steps 20 --warmup 5 \
  > gpurun_out/r2h_bench_n4_star_e2e.json 2> gpurun_out/r2h_bench_n4_star_e2e.err
timeout 900 $TR --nproc-per-node 4 --master-port 29972 tools/c4_sweep.py gpurun_out/r2h_c4_sweep_n4.jsonl > gpurun_out/r2h_c4_sweep_n4.log 2>&1
timeout 900 $TR --nproc-per-node 2 --master-port 29974 tools/c4_sweep.py gpurun_out/r2h_c4_sweep_n2.jsonl > gpurun_out/r2h_c4_sweep_n2.log 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r2h_pytest_mg.log 2>&1; echo rc=$? >> gpurun_out/r2h_pytest_mg.log
timeout 1500 $TR --nproc-per-node 4 --master-port 29981 tools/calibrate_peer.py gpurun_out/calg > gpurun_out/r2h_cal_n4.log 2>&1
timeout 1500 $TR --nproc-per-node 2 --master-port 29982 tools/calibrate_peer.py gpurun_out/calg > gpurun_out/r2h_cal_n2.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 1500 bash tools/nvlink_profile.sh 2 > gpurun_out/r2h_nvl.log 2>&1
