export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for a in ring tree; do
  timeout 300 $TR --nproc-per-node 4 --master-port 29954 bench.py --gpus 4 --algo $a --no-e2e > gpurun_out/r2ring5_bench_n4_$a.json 2>/dev/null
done
timeout 300 $TR --nproc-per-node 4 --master-port 29955 bench.py --gpus 4 --mode var --no-e2e > gpurun_out/r2ring5_bench_n4_var.json 2>/dev/null
timeout 300 $TR --nproc-per-node 4 --master-port 29814 tools/diag_mp_timeline.py star ring > gpurun_out/r2ring5_tl_n4_ring.txt 2>&1
timeout 900 $TR --nproc-per-node 4 --master-port 29961 tools/soak_mp.py 200003 1500 50 > gpurun_out/r2ring5_soak_n4.log 2>&1; echo rc=$? >> gpurun_out/r2ring5_soak_n4.log
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r2ring5_pytest_mg.log 2>&1; echo rc=$? >> gpurun_out/r2ring5_pytest_mg.log
