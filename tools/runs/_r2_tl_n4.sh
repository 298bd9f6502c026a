# 4-GPU: per-rank timelines of STAR ring / tree (in-place aggregate), NVLink
# bytes per step from the NVML counters, bench lines of the merged in-place kernel
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 2; do
  for a in ring tree; do
    timeout 300 $TR --nproc-per-node $N --master-port 2981$N tools/diag_mp_timeline.py star $a > gpurun_out/r2l_tl_n${N}_$a.txt 2>&1
  done
  timeout 600 $TR --nproc-per-node $N --master-port 2982$N tools/nvlink_bytes.py gpurun_out/r2l_nvlink_bytes_n$N.json > gpurun_out/r2l_nvlink_n$N.log 2>&1
  for cfg in "star ring" "star tree" "var ring"; do
    set -- $cfg
    timeout 300 $TR --nproc-per-node $N --master-port 2995$N bench.py --gpus $N --mode $1 --algo $2 --no-e2e \
      > gpurun_out/r2l_bench_n${N}_$1_$2.json 2> gpurun_out/r2l_bench_n${N}_$1_$2.err
  done
done
