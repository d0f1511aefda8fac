"""Per-source-function breakdown of an ncu report, using the source embedded
in the report (--import-source on), so it stays valid after the sources change.

usage: ncu_src.py report.ncu-rep [kernel-substring] [top-lines]
prints warp-instruction %, thread-instruction %, stall-sample % and the
long-scoreboard share per enclosing function, then the top lines by stalls.
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", *args],
                          capture_output=True, text=True).stdout


# full source text per file -> function start lines
full = ncu("--print-source", "cuda")
starts = collections.defaultdict(list)
fname = None
pat = re.compile(r"^(?:template <[^>]*>\s*)?(?:static\s+)?(?:__host__\s+)?(?:__device__|__global__)[^(]*?\b(\w+)\s*\(")
for row in csv.reader(io.StringIO(full)):
    if len(row) >= 2 and row[0] in ("File Name", "File Path"):
        fname = row[1].split("/")[-1]
        continue
    if fname and len(row) >= 2 and row[0].isdigit():
        ln, src = int(row[0]), row[1]
        m = pat.match(src)
        name = None
        if m and m.group(1) != "__launch_bounds__":
            name = m.group(1)
        elif re.match(r"^\s+(k_\w+)\(", src):
            name = src.strip().split("(")[0]
        elif m:
            mm = re.search(r"\)\s+(\w+)\(", src)
            if mm:
                name = mm.group(1)
        if name:
            starts[fname].append((ln, name))


# headers the report did not embed: read the current file (valid while unchanged)
import os
_csrc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2112_05570_b200", "csrc")
for _f in os.listdir(_csrc):
    if _f.endswith((".cuh", ".cu")) and _f not in starts:
        for _k, _src in enumerate(open(os.path.join(_csrc, _f)).read().splitlines(), 1):
            _m = pat.match(_src)
            if _m and _m.group(1) != "__launch_bounds__":
                starts[_f].append((_k, _m.group(1)))


def func_of(f, ln):
    name = f
    for k, n in starts.get(f, []):
        if k <= ln:
            name = n
    return name


out = ncu("--print-source", "cuda,sass")
agg = collections.defaultdict(lambda: [0, 0, 0, 0])
lines = collections.defaultdict(lambda: [0, 0, 0, 0, ""])
fname, kern, hdr = None, "", None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        kern = row[1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0].isdigit() or (ksub and ksub not in kern):
        continue
    try:
        wi = int(row[hdr.index("Instructions Executed")] or 0)
        ti = int(row[hdr.index("Thread Instructions Executed")] or 0)
        ss = int(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        ls = int(row[hdr.index("stall_long_sb")] or 0)
    except (ValueError, IndexError):
        continue
    fn = func_of(fname, int(row[0]))
    a = agg[fn]
    a[0] += wi; a[1] += ti; a[2] += ss; a[3] += ls
    L = lines[(fname, int(row[0]))]
    L[0] += wi; L[1] += ti; L[2] += ss; L[3] += ls; L[4] = row[1].strip()[:60]

T = [sum(v[i] for v in agg.values()) or 1 for i in range(4)]
print(f"warp-inst {T[0]}  thread-inst {T[1]}  stall samples {T[2]}  long_sb {T[3]}")
print(f"{'function':32s} {'warp%':>7s} {'thr%':>7s} {'stall%':>7s} {'lsb%':>7s} {'act/w':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
    act = v[1] / v[0] if v[0] else 0
    print(f"{k:32s} {100*v[0]/T[0]:7.2f} {100*v[1]/T[1]:7.2f} {100*v[2]/T[2]:7.2f} {100*v[3]/T[3]:7.2f} {act:6.1f}")
print()
print(f"{'line':24s} {'warp%':>7s} {'stall%':>7s} {'lsb%':>7s}  source")
for k, v in sorted(lines.items(), key=lambda x: -x[1][2])[:top]:
    print(f"{k[0]+':'+str(k[1]):24s} {100*v[0]/T[0]:7.2f} {100*v[2]/T[2]:7.2f} {100*v[3]/T[3]:7.2f}  {v[4]}")
