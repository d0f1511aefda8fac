"""Attribute an ncu report's per-SASS metrics to CUDA source lines.

usage: ncu_lines.py report.ncu-rep libmwt.so [kernel-substring] [top]
(the .so must be the exact build that was profiled)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, so = sys.argv[1], os.path.abspath(sys.argv[2])
ksub = sys.argv[3] if len(sys.argv) > 3 else "k_trace"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
kname = rows[0][1]
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
recs = []
for row in rows[2:]:
    try:
        a = int(row[ix["Address"]], 16)
    except ValueError:
        continue
    recs.append((a, row[ix["Source"]].strip(), int(row[ix["Instructions Executed"]] or 0),
                 int(row[ix["Thread Instructions Executed"]] or 0),
                 int(row[ix["Warp Stall Sampling (All Samples)"]] or 0)))
base = min(a for a, *_ in recs)
# mangled kernel name in the cubin
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, capture_output=True)
    text = ""
    for f in os.listdir(d):
        if f.endswith(".cubin"):
            text += subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, f)], capture_output=True,
                                   text=True).stdout
# find the function whose demangled name matches the profiled kernel
funcs = re.findall(r"\.text\.(\S+):\n", text)
cand = [f for f in funcs if ksub in subprocess.run(["c++filt", f], capture_output=True, text=True).stdout]
want = None
norm = re.sub(r"\(bool\)1", "true", re.sub(r"\(bool\)0", "false", kname))
norm = re.sub(r"\(int\)(-?\d+)", r"\1", norm).replace(" ", "")
for f in cand:
    dem = subprocess.run(["c++filt", f], capture_output=True, text=True).stdout.strip().replace(" ", "")
    if dem.split("(")[0] == norm.split("(")[0]:
        want = f
if want is None:
    raise SystemExit(f"no SASS function matches {kname!r}")
body = text.split(f".text.{want}:\n", 1)[1].split("//---------------------", 1)[0]
linemap = {}
cur = None
for ln in body.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        linemap[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: [0, 0, 0])
for a, s, wi, ti, sm in recs:
    k = linemap.get(a - base, "?")
    agg[k][0] += wi
    agg[k][1] += ti
    agg[k][2] += sm
T = sum(v[1] for v in agg.values())
S = sum(v[2] for v in agg.values())
W = sum(v[0] for v in agg.values())
print(f"{kname[:100]}\n warp-inst {W}  thread-inst {T}  stall samples {S}")
print(f"{'line':28s} {'warp-inst%':>10s} {'thr-inst%':>10s} {'stall%':>8s} {'act/warp':>8s}")
for k, (wi, ti, sm) in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
    print(f"{k:28s} {100*wi/W:10.2f} {100*ti/T:10.2f} {100*sm/S:8.2f} {ti/max(wi,1):8.1f}")
