"""Group ncu per-line metrics (tools/ncu_lines.py machinery) into source regions."""
import collections
import os
import re
import subprocess
import sys

sys.argv += [] if len(sys.argv) > 3 else ["k_trace"]
rep, so, ksub = sys.argv[1], os.path.abspath(sys.argv[2]), sys.argv[3]
out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ncu_lines.py"), rep, so, ksub,
                      "100000"], capture_output=True, text=True).stdout
regions = [  # (file, first line, last line, name)
    ("mwt_device.cuh", 152, 229, "raygen (mix64/u01/gen_ray)"),
    ("mwt_device.cuh", 231, 234, "sa2 (locate contains)"),
    ("mwt_device.cuh", 236, 240, "side_of (walk)"),
    ("mwt_device.cuh", 242, 292, "rsi + canonical (epilogue)"),
    ("mwt_device.cuh", 293, 296, "pick"),
    ("mwt_device.cuh", 297, 310, "load_ray"),
    ("mwt_walk.cu", 30, 56, "corners/edge_areas"),
    ("mwt_walk.cu", 57, 129, "brute/flood"),
    ("mwt_walk.cu", 130, 194, "locate"),
    ("mwt_walk.cu", 203, 262, "walk_first/load_step"),
    ("mwt_walk.cu", 263, 290, "walk_general"),
    ("mwt_walk.cu", 291, 344, "walk_step"),
    ("mwt_walk.cu", 345, 402, "terminal"),
    ("mwt_walk.cu", 403, 431, "hist"),
    ("mwt_walk.cu", 432, 515, "prologue glue"),
    ("mwt_walk.cu", 516, 601, "k_trace loop"),
    ("mwt_walk.cu", 602, 747, "k_trace_q loop"),
]
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for ln in out.splitlines():
    m = re.match(r"(\S+):(\d+)\s+([\d.]+)\s+([\d.]+)\s+([\d.]+)", ln)
    if not m:
        continue
    f, l = m.group(1), int(m.group(2))
    name = next((r[3] for r in regions if r[0] == f and r[1] <= l <= r[2]), f"other {f}")
    for k in range(3):
        agg[name][k] += float(m.group(3 + k))
print(out.splitlines()[0])
print(f"{'region':34s} {'warp%':>7s} {'thr%':>7s} {'stall%':>7s}  thr/warp")
for name, (w, t, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{name:34s} {w:7.2f} {t:7.2f} {s:7.2f}")
