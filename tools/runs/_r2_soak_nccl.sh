export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
FC_NO_P2P=1 timeout 900 $TR --nproc-per-node 4 --master-port 29963 tools/soak_mp.py 200003 600 50 > gpurun_out/r2soak3_n4_nccl.log 2>&1; echo rc=$? >> gpurun_out/r2soak3_n4_nccl.log
timeout 900 $TR --nproc-per-node 4 --master-port 29961 tools/soak_mp.py 200003 1500 50 > gpurun_out/r2soak3_n4.log 2>&1; echo rc=$? >> gpurun_out/r2soak3_n4.log
