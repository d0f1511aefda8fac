"""Group ncu per-line metrics (tools/ncu_lines.py) by the enclosing source
function (derived from the current csrc sources)."""
import collections
import os
import re
import subprocess
import sys

rep, so = sys.argv[1], os.path.abspath(sys.argv[2])
ksub = sys.argv[3] if len(sys.argv) > 3 else "k_trace"
csrc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_2112_05570_b200", "csrc")
starts = {}  # file -> [(line, name)]
pat = re.compile(r"^(?:template <[^>]*>\s*)?(?:static\s+)?(?:__host__\s+)?(?:__device__|__global__)[^(]*?\b(\w+)\s*\(")
for f in os.listdir(csrc):
    if not f.endswith((".cu", ".cuh")):
        continue
    lines = open(os.path.join(csrc, f)).read().splitlines()
    lst = []
    for k, ln in enumerate(lines, 1):
        m = pat.match(ln)
        if m and m.group(1) != "__launch_bounds__":
            lst.append((k, m.group(1)))
        elif re.match(r"^\s+k_trace(_q)?\(", ln):
            lst.append((k - 1, ln.strip().split("(")[0]))
        elif m:
            mm = re.search(r"\)\s+(\w+)\(", ln)
            if mm:
                lst.append((k, mm.group(1)))
    starts[f] = lst
out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ncu_lines.py"), rep, so, ksub,
                      "100000"], capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for ln in out.splitlines():
    m = re.match(r"(\S+):(\d+)\s+([\d.]+)\s+([\d.]+)\s+([\d.]+)", ln)
    if not m:
        continue
    f, l = m.group(1), int(m.group(2))
    name = f
    for k, n in starts.get(f, []):
        if k <= l:
            name = f"{n} ({f})"
    for i in range(3):
        agg[name][i] += float(m.group(3 + i))
print(out.splitlines()[0] if out else "no output")
print(f"{'function':44s} {'warp%':>7s} {'thr%':>7s} {'stall%':>7s}")
for name, (w, t, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    if w >= 0.05 or s >= 0.05:
        print(f"{name:44s} {w:7.2f} {t:7.2f} {s:7.2f}")
