# compute-sanitizer memcheck over a 2-rank peer-exchange soak (2 GPUs)
OUT=gpurun_out/sanitize
mkdir -p $OUT
export OMP_NUM_THREADS=1
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --target-processes all --print-limit 50 \
  --error-exitcode 9 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29931 tools/soak_mp.py 60001 30 10 > $OUT/memcheck_soak_n2.log 2>&1
echo "exit=$?" >> $OUT/memcheck_soak_n2.log
tail -5 $OUT/memcheck_soak_n2.log
