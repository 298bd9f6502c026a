for r in a b c; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2l2pf_bench_$r.json 2>/dev/null
done
timeout 300 python tools/diag_select.py > gpurun_out/r2l2pf_sel.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2l2pf_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2l2pf_pytest.log
