export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  for cfg in "star ring" "star tree" "var ring"; do
    set -- $cfg
    timeout 300 $TR --nproc-per-node $N --master-port 2995$N bench.py --gpus $N --mode $1 --algo $2 --no-e2e > gpurun_out/r2pe_bench_n${N}_$1_$2.json 2>/dev/null
  done
done
timeout 900 $TR --nproc-per-node 4 --master-port 29961 tools/soak_mp.py 200003 1500 50 > gpurun_out/r2pe_soak_n4.log 2>&1; echo rc=$? >> gpurun_out/r2pe_soak_n4.log
timeout 900 $TR --nproc-per-node 2 --master-port 29962 tools/soak_mp.py 200003 1500 50 > gpurun_out/r2pe_soak_n2.log 2>&1; echo rc=$? >> gpurun_out/r2pe_soak_n2.log
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r2pe_pytest_mg.log 2>&1; echo rc=$? >> gpurun_out/r2pe_pytest_mg.log
timeout 300 $TR --nproc-per-node 2 --master-port 29816 tools/diag_mp_timeline.py star ring > gpurun_out/r2pe_tl_n2_ring.txt 2>&1
