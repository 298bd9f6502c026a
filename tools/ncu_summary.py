"""Summarise `ncu --set full` reports of the step's kernels into one JSON
(profiles/): per captured launch, the kernel, duration, DRAM bytes
read/written, DRAM throughput, registers, launch shape.
Usage: python tools/ncu_summary.py out.json report.ncu-rep [report2 ...]"""
import csv
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    return [{h[i]: (v[i], u[i]) for i in range(len(h))} for v in rows[2:]], out


res = []
for rep in sys.argv[2:]:
    rs, text = rows_of(rep)
    with open(sys.argv[1].replace(".json", "_raw.csv"), "a") as f:
        f.write(text)
    for r in rs:
        g = lambda m: float(r[m][0].replace(",", ""))
        res.append({
            "kernel": r["Kernel Name"][0].split("(")[0],
            "duration_us": g("gpu__time_duration.sum") / (1e3 if r["gpu__time_duration.sum"][1] == "ns" else 1),
            "dram_read_bytes": g("dram__bytes_read.sum") * SCALE.get(r["dram__bytes_read.sum"][1], 1),
            "dram_write_bytes": g("dram__bytes_write.sum") * SCALE.get(r["dram__bytes_write.sum"][1], 1),
            "dram_throughput_pct_of_peak": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "registers": int(g("launch__registers_per_thread")),
            "grid": int(g("launch__grid_size")),
            "block": int(g("launch__block_size")),
        })
json.dump({"reports": sys.argv[2:], "kernels": res}, open(sys.argv[1], "w"), indent=1)
print(json.dumps(res, indent=1))
