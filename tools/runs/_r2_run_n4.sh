export OMP_NUM_THREADS=1
nvidia-smi topo -m > gpurun_out/r2_topo_n4.txt 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r2_pytest_n4_mg.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest_n4_mg.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 tools/calibrate_peer.py gpurun_out/cal_n4 > gpurun_out/r2_cal_n4.log 2>&1
for cfg in "star ring" "star tree" "ag ring" "dense ring" "var ring"; do
  set -- $cfg
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 4 --mode $1 --algo $2 --no-e2e > gpurun_out/r2_bench_n4_$1_$2.json 2> gpurun_out/r2_bench_n4_$1_$2.err
done
for cfg in "dense ring" "star ring" "ag ring"; do
  set -- $cfg
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29813 bench.py --gpus 2 --mode $1 --algo $2 --no-e2e > gpurun_out/r2_bench_n2_$1_$2.json 2> gpurun_out/r2_bench_n2_$1_$2.err
done
timeout 300 python tools/diag_select.py 138000000 0.01 > gpurun_out/r2_sel_n4box.txt 2>&1; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_n4box_n1.json 2>/dev/null
