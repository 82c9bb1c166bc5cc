"""Top SASS instructions by warp-stall samples from an ncu report (source page).

    python tools/ncu_hot.py report.ncu-rep kernel_regex [N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
rows = [x for x in r[2:] if len(x) == len(h) and x[0] != "Address"]
si = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
tot = sum(int(x[si] or 0) for x in rows)
print("total samples", tot, "instructions", len(rows))
order = sorted(range(len(rows)), key=lambda i: -int(rows[i][si] or 0))
for i in order[:n]:
    print(f"{rows[i][si]:>6} [{i:5d}] {rows[i][src].strip()[:90]}")
