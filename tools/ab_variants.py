"""A/B the walk-kernel variants on every config (diagnostic).

usage: python tools/ab_variants.py [log2 rays] [variants, comma-separated]
Prints ms and rays/s of the fused generated box-entry launch per config, mesh
and variant (1: global records, 2: default choice, 3: per-triangle table first).
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_05570_b200 import _lib  # noqa: E402
from paper_2112_05570_b200.engine import DeviceMesh, new_histogram  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 22
variants = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "2,3,1").split(",")]
n = 1 << lg
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for cfg in ("lines64", "lines1024", "grass4096", "hair512", "floorplan64"):
    box = (0.0, 0.0, 1.0, 0.5) if cfg.startswith("grass") else (0.0, 0.0, 1.0, 1.0)
    for which in ("mwt", "cdt"):
        d = os.path.join(ROOT, "fixtures", "data", cfg)
        mesh = DeviceMesh.from_files(os.path.join(d, "scene.txt"), os.path.join(d, f"{which}.tri"))
        hist = new_histogram()
        row = []
        for v in variants:
            _lib.check(_lib.lib.mwt_set_tuning(6, 4, v))
            ms = timeit(lambda: mesh.trace_generated_device(0, box, 0, 0, n, True, hist))
            row.append(f"v{v} {ms:.3f} ms {n / ms / 1e6:.2f}e9/s")
        _lib.check(_lib.lib.mwt_set_tuning(6, 4, 2))
        print(f"{cfg:12s} {which}  smem {mesh.info.walk_smem_bytes:7d}  " + "  |  ".join(row), flush=True)
