# final validation of the round's last code on a 2-GPU lease: the whole
# GPU suite (multi-GPU cases at N=2), smoke, the N=1 bench line
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2fin_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2fin_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2fin_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2fin_smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py > gpurun_out/r2fin_bench_n1.json 2> gpurun_out/r2fin_bench_n1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29952 bench.py --gpus 2 --no-e2e > gpurun_out/r2fin_bench_n2.json 2> gpurun_out/r2fin_bench_n2.err
