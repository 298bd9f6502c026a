"""Top SASS instructions by warp-stall samples from an ncu report's source page."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[2].isdigit()]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1
idx = {d["Address"]: i for i, d in enumerate(data)}
top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:n]
for d in top:
    i = idx[d["Address"]]
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    prev = data[i - 1]["Source"].strip() if i else ""
    print(f"{s / tot * 100:5.1f}%  {i:5d}  {d['Source'].strip()[:60]:60s} | prev: {prev[:50]}")
