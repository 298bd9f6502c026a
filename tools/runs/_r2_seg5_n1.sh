timeout 300 python tools/diag_segments.py > gpurun_out/r2w_segments.txt 2>&1
timeout 600 python tools/diag_select.py 355000000 0.1 > gpurun_out/r2w_sel_c4_cr01.txt 2>&1
