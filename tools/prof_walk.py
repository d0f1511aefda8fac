"""Launch the walk-only path (rays + start triangles given) for ncu. args: cfg mesh mode n refill minb"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_05570_b200 import _lib  # noqa: E402
from paper_2112_05570_b200.engine import DeviceMesh  # noqa: E402

cfg, which, mode, n = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
refill, minb = int(sys.argv[5]), int(sys.argv[6])
box = (0.0, 0.0, 1.0, 0.5) if cfg.startswith("grass") else (0.0, 0.0, 1.0, 1.0)
d = os.path.join(ROOT, "fixtures", "data", cfg)
mesh = DeviceMesh.from_files(os.path.join(d, "scene.txt"), os.path.join(d, f"{which}.tri"))
_lib.check(_lib.lib.mwt_set_tuning(refill, minb, int(os.environ.get("MWT_VARIANT", "0"))))
rays = mesh.raygen_device(mode, box, 0, 0, n)
tid, _ = mesh.locate_device(rays[:, :2].contiguous())
for _ in range(4):
    out = mesh.trace_device(rays, tid, want=("seg", "t", "steps"))
torch.cuda.synchronize()
print("ok", float(out["steps"].double().mean()))
