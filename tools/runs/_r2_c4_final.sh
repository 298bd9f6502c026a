export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29972 tools/c4_sweep.py gpurun_out/r2c4_sweep_n4.jsonl > gpurun_out/r2c4_sweep_n4.log 2>&1
timeout 900 $TR --nproc-per-node 2 --master-port 29974 tools/c4_sweep.py gpurun_out/r2c4_sweep_n2.jsonl > gpurun_out/r2c4_sweep_n2.log 2>&1
