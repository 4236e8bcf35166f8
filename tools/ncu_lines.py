"""Per-source-line stall samples / instructions of one kernel in an ncu
report: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hdr]
si, ni = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[hdr + 1:]:
    if len(r) < len(h) or r[0] == "":
        continue
    try:
        data.append((float(r[si]), float(r[ni]), r[0], r[1][:110]))
    except ValueError:
        pass
ts = sum(d[0] for d in data) or 1
tn = sum(d[1] for d in data) or 1
print(f"samples {ts:.0f}, instructions {tn:.0f}")
for d in sorted(data, reverse=True)[:top]:
    print(f"{100 * d[0] / ts:5.1f}% {100 * d[1] / tn:5.1f}% {d[2]:>4} {d[3]}")
