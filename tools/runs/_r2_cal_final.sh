# last multi-GPU run: AG lines and e2e at N=4, NVLink calibration at N=4 and N=2
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out/calj
for N in 4 2; do
  timeout 300 $TR --nproc-per-node $N --master-port 2995$N bench.py --gpus $N --mode ag --no-e2e > gpurun_out/r2cj_bench_n${N}_ag_ring.json 2>/dev/null
done
timeout 300 $TR --nproc-per-node 4 --master-port 29971 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2cj_bench_n4_star_e2e.json 2>/dev/null
timeout 1200 $TR --nproc-per-node 4 --master-port 29981 tools/calibrate_peer.py gpurun_out/calj > gpurun_out/r2cj_cal_n4.log 2>&1
timeout 900 $TR --nproc-per-node 2 --master-port 29982 tools/calibrate_peer.py gpurun_out/calj > gpurun_out/r2cj_cal_n2.log 2>&1
