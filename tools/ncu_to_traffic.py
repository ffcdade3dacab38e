"""Summarise one `ncu --set full` capture of a config's dominant kernel into
profiles/ncu_traffic_<config>.json (read by bench.py for roofline.traffic).

    python tools/ncu_to_traffic.py REPORT.ncu-rep CONFIG N_LOCAL ALG_BYTES_PER_LAUNCH
"""
import csv
import json
import os
import subprocess
import sys

rep, cfg, n, alg = sys.argv[1], sys.argv[2], int(sys.argv[3]), float(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
m = dict(zip(h, v))
units = dict(zip(h, u))


def val(k):
    x = float(m[k].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "usecond": 1,
             "us": 1, "nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}.get(units.get(k, ""), 1)
    return x * scale


rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
res = {
    "kernel": m.get("Kernel Name", "")[:120],
    "n": n,
    "dram_bytes_per_launch": rd + wr,
    "dram_read": rd,
    "dram_write": wr,
    "algorithmic_bytes": alg,
    "traffic_over_algorithmic": round((rd + wr) / alg, 4),
    "duration_us_ncu": val("gpu__time_duration.sum"),
    "issue_active_pct": float(m["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
    "dram_throughput_pct": float(m["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
    "registers": int(float(m["launch__registers_per_thread"])),
    "warps_active_per_sm": float(m["sm__warps_active.avg.per_cycle_active"]),
    "source": f"{os.path.basename(rep)} (ncu --set full --clock-control none, one launch inside bench.py --config {cfg})",
}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                    f"ncu_traffic_{cfg}.json")
with open(path, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res))
