# one compute-sanitizer tool over tools/sanitize_case.py (one GPU):
#   bash tools/sanitize_one.sh memcheck|racecheck|synccheck|initcheck
T=$1
OUT=gpurun_out/sanitize
mkdir -p $OUT
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool $T --print-limit 50 --error-exitcode 9 \
  python tools/sanitize_case.py > $OUT/$T.log 2>&1
echo "exit=$?" >> $OUT/$T.log
tail -5 $OUT/$T.log
