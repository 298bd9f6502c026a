"""Top source lines by warp-stall samples from `ncu -i X --page source --csv
--print-source cuda,sass` output (stdin or a file): line, samples, the
dominant stall reasons.  Usage: python tools/ncu_source_top.py dump.csv [N]"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows, hdr, fname = [], None, ""
with open(path, newline="") as f:
    for r in csv.reader(f):
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[0]:
            continue
        d = dict(zip(hdr, r))
        try:
            n = int(d["Warp Stall Sampling (All Samples)"])
        except ValueError:
            continue
        stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
        rows.append((n, f"{fname}:{r[0]}", r[1][:90], sorted(stalls.items(), key=lambda x: -x[1])[:3]))
tot = sum(x[0] for x in rows)
print(f"total samples {tot}")
for n, loc, src, st in sorted(rows, key=lambda x: -x[0])[:top]:
    print(f"{n:7d} {100.0 * n / max(tot, 1):5.1f}% {loc:24} {src:90} {st}")
