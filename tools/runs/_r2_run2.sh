set -x
export OMP_NUM_THREADS=1
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/r2_pytest2.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/calibrate_peer.py gpurun_out/cal > gpurun_out/r2_cal_n2.log 2>&1
for m in star ag dense; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --mode $m > gpurun_out/r2_bench_n2_$m.json 2> gpurun_out/r2_bench_n2_$m.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --mode star --algo tree > gpurun_out/r2_bench_n2_startree.json 2> gpurun_out/r2_bench_n2_startree.err
