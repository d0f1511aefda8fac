"""Median time of the fused trace (mwt_trace_generated_dev) per config / ray
part / generator order at the BASELINE sizes, L2 flushed before each run; one
JSON line.  For A/B of library builds: MWT_LIB_PATH=... python tools/time_fused.py cfg ..."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2112_05570_b200.engine import DeviceMesh  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
for cfg in sys.argv[1:] or ["floorplan64", "lines1024"]:
    box, parts = bench.CONFIGS[cfg]
    m = DeviceMesh.from_files(*bench.fixture(cfg, "mwt"))
    for order in ("coherent", "iid"):
        for base, n in parts:
            mw = bench.mode_word(base, order)
            ts = []
            for k in range(9):
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                m.trace_generated_device(mw, box, 0, 0, n, outputs=True, hist=None)
                b.record()
                torch.cuda.synchronize()
                if k >= 2:
                    ts.append(a.elapsed_time(b))
            out[f"{cfg}/{order}/{bench.part_name(base)}"] = round(float(np.median(ts)), 4)
print(json.dumps(out))
