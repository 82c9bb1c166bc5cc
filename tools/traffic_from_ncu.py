"""DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of ncu reports,
for bench.py's `traffic` fields (profiles/spmm_traffic.json, profiles/gram_traffic.json).

    python tools/traffic_from_ncu.py REPORT.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        def get(k):
            i = h.index(k)
            return float(v[i]) * UNITS.get(u[i], 1.0)
        res.append((get("dram__bytes_read.sum"), get("dram__bytes_write.sum"),
                    float(v[h.index("gpu__time_duration.sum")])))
    return res


for rep in sys.argv[1:]:
    for r, w, t in launches(rep):
        print(f"{rep}: read {r / 1e9:.3f} GB  write {w / 1e9:.3f} GB  total {int(r + w)} B  time {t}")
