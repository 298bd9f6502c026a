# compute-sanitizer over the path's kernels (one GPU) and over the peer
# exchange (2 ranks).  Logs in gpurun_out/sanitize/.
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_case.py > $OUT/$tool.log 2>&1
  echo "exit=$?" >> $OUT/$tool.log
done
if [ "$(nvidia-smi -L | wc -l)" -ge 2 ]; then
  timeout 1200 $CS --tool memcheck --target-processes all --print-limit 50 --error-exitcode 9 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
    tools/soak_mp.py 60001 40 10 > $OUT/memcheck_soak_n2.log 2>&1
  echo "exit=$?" >> $OUT/memcheck_soak_n2.log
  timeout 1200 $CS --tool synccheck --target-processes all --print-limit 50 --error-exitcode 9 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 \
    tools/soak_mp.py 60001 20 10 > $OUT/synccheck_soak_n2.log 2>&1
  echo "exit=$?" >> $OUT/synccheck_soak_n2.log
fi
