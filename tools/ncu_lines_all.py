"""Every source line of a kernel with executed warp instructions, in source
order, as warp instructions per 32 rays (per-ray fixed costs at a glance).
usage: ncu_lines_all.py report.ncu-rep kernel-substring rays [min-per-32-rays]"""
import collections
import csv
import io
import subprocess
import sys

rep, ksub, rays = sys.argv[1], sys.argv[2], int(sys.argv[3])
lo = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines = collections.defaultdict(lambda: [0, 0, ""])
fname, kern, hdr = None, "", None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] in ("File Path", "File Name"):
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        kern = row[1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0].isdigit() or (ksub and kern and ksub not in kern):
        continue
    try:
        wi = int(row[hdr.index("Instructions Executed")] or 0)
        ss = int(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    L = lines[(fname, int(row[0]))]
    L[0] += wi; L[1] += ss; L[2] = row[1].rstrip()[:90]
warps = rays / 32.0
tot = sum(v[0] for v in lines.values())
print(f"total {tot / warps:.1f} warp instructions per 32 rays")
for k in sorted(lines):
    v = lines[k]
    if v[0] / warps >= lo:
        print(f"{k[0]:>14s}:{k[1]:<5d} {v[0] / warps:7.1f}  {v[2]}")
