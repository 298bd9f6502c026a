"""Host<->device copy bandwidth of this box (the floor of bench.py's e2e):
pinned 552 MB buffers (config 3's gradient), H2D alone, D2H alone, and both
directions at once on two streams, CUDA-event timed.
Usage: python tools/diag_pcie.py [bytes]"""
import json
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 552_000_000
h_up = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_dn = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_up = torch.empty(n, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def up():
    d_up.copy_(h_up, non_blocking=True)


def down():
    h_dn.copy_(d_dn, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        d_up.copy_(h_up, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dn.copy_(d_dn, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


out = {"bytes": n}
for name, fn in (("h2d", up), ("d2h", down), ("both", both)):
    ms = timed(fn)
    out[name + "_ms"] = round(ms, 3)
    out[name + "_GBps"] = round((2 if name == "both" else 1) * n / ms / 1e6, 1)
print(json.dumps(out))
