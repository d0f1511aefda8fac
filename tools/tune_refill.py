"""Sweep the walk kernel's runtime knobs on the headline workload (diagnostic).

usage: [ORDER=coherent|iid] [N=rays] python tools/tune_refill.py [config] [min_blocks,...] [refill,...]
-- prints ms of the fused generated box-entry launch (default 2^24 coherent
rays, L2 flushed) per (refill_below, min_blocks)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2112_05570_b200 import _lib  # noqa: E402
from paper_2112_05570_b200.engine import DeviceMesh, new_histogram  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "lines1024"
d = os.path.join(ROOT, "fixtures", "data", cfg)
mesh = DeviceMesh.from_files(os.path.join(d, "scene.txt"), os.path.join(d, "mwt.tri"))
box = (0.0, 0.0, 1.0, 0.5) if cfg.startswith("grass") else (0.0, 0.0, 1.0, 1.0)
n = int(os.environ.get("N", 1 << 24))
MW = bench.mode_word(0, os.environ.get("ORDER", "coherent"))
hist = new_histogram()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(reps=15):
    for _ in range(3):
        mesh.trace_generated_device(MW, box, 0, 0, n, True, hist)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mesh.trace_generated_device(MW, box, 0, 0, n, True, hist)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for minb in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,3").split(",")]:
    for rb in [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "3,4,5,6,7,8,10").split(",")]:
        _lib.check(_lib.lib.mwt_set_tuning(rb, minb, 2))
        print(f"{cfg} min_blocks {minb} refill_below {rb:2d}: {timeit():.4f} ms", flush=True)
_lib.check(_lib.lib.mwt_set_tuning(6, 4, 2))
