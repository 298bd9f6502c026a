"""Summarise `ncu --set full` reports of the step's kernels into one JSON
(profiles/): duration, DRAM bytes read/written, DRAM throughput, registers,
launch shape.  Usage: python tools/ncu_summary.py out.json name=report.ncu-rep ..."""
import csv
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}, out


res = {}
for arg in sys.argv[2:]:
    name, rep = arg.split("=", 1)
    r, text = raw(rep)
    g = lambda m: float(r[m][0].replace(",", ""))
    res[name] = {
        "duration_us": g("gpu__time_duration.sum"),
        "dram_read_bytes": g("dram__bytes_read.sum") * SCALE[r["dram__bytes_read.sum"][1]],
        "dram_write_bytes": g("dram__bytes_write.sum") * SCALE[r["dram__bytes_write.sum"][1]],
        "dram_throughput_pct_of_peak": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "registers": int(g("launch__registers_per_thread")),
        "grid": int(g("launch__grid_size")),
        "block": int(g("launch__block_size")),
    }
    with open(sys.argv[1].replace(".json", f"_{name}_raw.csv"), "w") as f:
        f.write(text)
json.dump({"capture": "ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 3 -c 1 "
                      "python tools/profile_step.py (138M fp32, CR 0.01, STAR, world-1 NCCL context)",
           "kernels": res}, open(sys.argv[1], "w"), indent=1)
print(json.dumps(res, indent=1))
