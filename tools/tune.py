"""Sweep the persistent-walk tuning knobs on the GPU (diagnostic)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_05570_b200 import _lib  # noqa: E402
from paper_2112_05570_b200.engine import DeviceMesh, new_histogram, summarize_histogram  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "lines1024"
which = sys.argv[2] if len(sys.argv) > 2 else "mwt"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 24
box = (0.0, 0.0, 1.0, 0.5) if cfg.startswith("grass") else (0.0, 0.0, 1.0, 1.0)
d = os.path.join(ROOT, "fixtures", "data", cfg)
if not os.path.exists(os.path.join(d, f"{which}.tri")):
    which = "cdt"
mesh = DeviceMesh.from_files(os.path.join(d, "scene.txt"), os.path.join(d, f"{which}.tri"))
hist = new_histogram()
res = []
combos = [(0, 2, 0)] + [(r, m, 1) for m in (2, 3, 4) for r in (2, 4, 8)]
for refill, minb, variant in combos:
    if True:
        _lib.lib.mwt_set_tuning(refill, minb, variant)
        for mode in (0, 1):
            for _ in range(3):
                mesh.trace_generated_device(mode, box, 0, 0, n, outputs=True, hist=hist)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            times = []
            for _ in range(5):
                hist.zero_()
                e0.record()
                mesh.trace_generated_device(mode, box, 0, 0, n, outputs=True, hist=hist)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            h = summarize_histogram(hist)
            ms = float(np.median(times))
            res.append(dict(variant=variant, minb=minb, refill=refill, mode=mode, ms=ms, grays=n / ms / 1e6,
                            steps=h["steps_per_ray"], gbs=h["steps_sum"] * 32 / ms / 1e6))
            print(json.dumps(res[-1]), flush=True)
_lib.lib.mwt_set_tuning(4, 3, 1)
