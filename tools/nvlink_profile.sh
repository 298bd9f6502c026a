# NVLink byte counters of the peer-exchange kernels: rank 0 under ncu (only
# the exchange kernels, metrics-only), the other ranks plain.
#   bash tools/nvlink_profile.sh N
N=${1:-2}
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29791 WORLD_SIZE=$N OMP_NUM_THREADS=1
for r in $(seq 1 $((N - 1))); do
  RANK=$r LOCAL_RANK=$r python tools/nvl_case.py > gpurun_out/nvl_rank$r.log 2>&1 &
done
RANK=0 LOCAL_RANK=0 timeout 1500 ncu --clock-control none \
  --metrics nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:"k_fetch_gather|k_collect_packs|k_reduce_slice|k_reduce_root|k_decode_ar|k_agg_write" --csv \
  --log-file gpurun_out/nvl_n${N}_rank0.csv python tools/nvl_case.py > gpurun_out/nvl_rank0.log 2>&1
wait
