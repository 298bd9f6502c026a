timeout 1500 python -m pytest tests/test_multigpu.py -q > gpurun_out/r2fin_pytest_mg.log 2>&1; echo rc=$? >> gpurun_out/r2fin_pytest_mg.log
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_multigpu.py > gpurun_out/r2fin_pytest_gpu_rest.log 2>&1; echo rc=$? >> gpurun_out/r2fin_pytest_gpu_rest.log
