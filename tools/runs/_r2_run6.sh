export OMP_NUM_THREADS=1
timeout 300 python tools/diag_select.py 138000000 0.01 > gpurun_out/r2_sel6_c3.txt 2>&1
timeout 900 python -m pytest tests/test_multigpu.py tests/test_cpp_facade.py -x -q > gpurun_out/r2_pytest6_mg.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest6_mg.log
(cd tests/cpp && timeout 300 ./bench_facade 138000000 5) > gpurun_out/r2_bench_facade.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/calibrate_peer.py gpurun_out/cal6 > gpurun_out/r2_cal6_n2.log 2>&1
for m in star ag; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --mode $m --no-e2e > gpurun_out/r2_bench6_n2_$m.json 2> gpurun_out/r2_bench6_n2_$m.err
done
