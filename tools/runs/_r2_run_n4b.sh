export OMP_NUM_THREADS=1
timeout 300 python tools/diag_select.py 138000000 0.01 > gpurun_out/r2_sel9_c3.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench9_n1.json 2> gpurun_out/r2_bench9_n1.err
timeout 1500 python -m pytest tests/test_multigpu.py -x -q -k "peer_only or timeout or nccl_parity" > gpurun_out/r2_pytest9_mg.log 2>&1; echo rc=$? >> gpurun_out/r2_pytest9_mg.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29911 tools/calibrate_peer.py gpurun_out/cal9 > gpurun_out/r2_cal9_n4.log 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29912 tools/calibrate_peer.py gpurun_out/cal9 > gpurun_out/r2_cal9_n2.log 2>&1
