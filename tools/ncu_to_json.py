"""Extracts per-kernel DRAM traffic / pipe utilisation from an ncu --set full report
into profiles/ncu_kernel_metrics.json (read by bench.py for roofline.traffic)."""
import csv
import json
import os
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}


def num(r, k):
    try:
        return float(r[col[k]])
    except Exception:
        return None


res = json.load(open(out)) if os.path.exists(out) else {}
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", "").strip()
    rd, wr = num(r, "dram__bytes_read.sum"), num(r, "dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(units[col["dram__bytes_read.sum"]], 1)
    wr *= scale.get(units[col["dram__bytes_write.sum"]], 1)
    res[name] = {
        "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
        "duration_us": num(r, "gpu__time_duration.sum") * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(
            units[col["gpu__time_duration.sum"]], 1.0),
        "tensor_pipe_pct": num(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": num(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "fma_pipe_pct": num(r, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "alu_pipe_pct": num(r, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        "source": os.path.basename(rep),
    }
json.dump(res, open(out, "w"), indent=1, sort_keys=True)
print(json.dumps(res, indent=1))
