# final N=4 lines, calibration and C4 sweep after the ART-Ring changes
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out/cali
for cfg in "star ring" "star tree" "var ring" "ag ring"; do
  set -- $cfg
  timeout 300 $TR --nproc-per-node 4 --master-port 29954 bench.py --gpus 4 --mode $1 --algo $2 --no-e2e \
    > gpurun_out/r2f5_bench_n4_$1_$2.json 2> gpurun_out/r2f5_bench_n4_$1_$2.err
done
FC_INCR_DIV=0 timeout 300 $TR --nproc-per-node 4 --master-port 29974 bench.py --gpus 4 --no-e2e > gpurun_out/r2f5_bench_n4_star_ring_densedecode.json 2>/dev/null
FC_NO_P2P=1 timeout 300 $TR --nproc-per-node 4 --master-port 29964 bench.py --gpus 4 --no-e2e > gpurun_out/r2f5_bench_n4_star_ring_nccl.json 2>/dev/null
timeout 300 $TR --nproc-per-node 4 --master-port 29971 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2f5_bench_n4_star_e2e.json 2>/dev/null
timeout 300 $TR --nproc-per-node 4 --master-port 29815 tools/diag_mp_timeline.py star tree > gpurun_out/r2f5_tl_n4_tree.txt 2>&1
timeout 1500 $TR --nproc-per-node 4 --master-port 29981 tools/calibrate_peer.py gpurun_out/cali > gpurun_out/r2f5_cal_n4.log 2>&1
timeout 900 $TR --nproc-per-node 4 --master-port 29972 tools/c4_sweep.py gpurun_out/r2f5_c4_sweep_n4.jsonl > gpurun_out/r2f5_c4_sweep_n4.log 2>&1
