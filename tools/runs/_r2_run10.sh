export OMP_NUM_THREADS=1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench10_n1.json 2> gpurun_out/r2_bench10_n1.err
timeout 1800 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r2_pytest10_mg.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest10_mg.log
for a in ring tree; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29921 bench.py --gpus 4 --mode star --algo $a --no-e2e > gpurun_out/r2_bench10_n4_star_$a.json 2> gpurun_out/r2_bench10_n4_star_$a.err
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29922 tools/calibrate_peer.py gpurun_out/cal10 > gpurun_out/r2_cal10_n4.log 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29923 tools/calibrate_peer.py gpurun_out/cal10 > gpurun_out/r2_cal10_n2.log 2>&1
