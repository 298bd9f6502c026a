import ctypes as C, sys
sys.path.insert(0, '.')
from paper_2312_02493_b200 import flexcomm as fc
from paper_2312_02493_b200._abi import check, lib
with fc.Cluster(1, 138_000_000, max_cr=0.1) as cl:
    cl.fill_synthetic(0, 42, 0, 0)
    out = []
    for w in (4, 5, 4, 5):
        m = C.c_double()
        check(lib.fc_diag_kernel_ms(cl._ctx, w, 10, C.byref(m)))
        out.append((w, round(m.value * 1e3, 1)))
    print(out)
