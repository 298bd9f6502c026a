export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r2gq_pytest_mg.log 2>&1; echo rc=$? >> gpurun_out/r2gq_pytest_mg.log
for N in 4 2; do
  for cfg in "star ring" "star tree" "var ring"; do
    set -- $cfg
    timeout 300 $TR --nproc-per-node $N --master-port 2995$N bench.py --gpus $N --mode $1 --algo $2 --no-e2e > gpurun_out/r2gq_bench_n${N}_$1_$2.json 2>/dev/null
  done
done
timeout 300 $TR --nproc-per-node 4 --master-port 29814 tools/diag_mp_timeline.py star ring > gpurun_out/r2gq_tl_n4_ring.txt 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29815 tools/diag_mp_timeline.py star tree > gpurun_out/r2gq_tl_n4_tree.txt 2>&1
timeout 900 $TR --nproc-per-node 4 --master-port 29961 tools/soak_mp.py 200003 1500 50 > gpurun_out/r2gq_soak_n4.log 2>&1; echo rc=$? >> gpurun_out/r2gq_soak_n4.log
