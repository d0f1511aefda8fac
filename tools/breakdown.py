"""Time the pieces of the hot path separately (diagnostic)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_05570_b200 import _lib  # noqa: E402
from paper_2112_05570_b200.engine import DeviceMesh, new_histogram  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "lines1024"
which = sys.argv[2] if len(sys.argv) > 2 else "cdt"
n = 1 << 24
box = (0.0, 0.0, 1.0, 0.5) if cfg.startswith("grass") else (0.0, 0.0, 1.0, 1.0)
d = os.path.join(ROOT, "fixtures", "data", cfg)
mesh = DeviceMesh.from_files(os.path.join(d, "scene.txt"), os.path.join(d, f"{which}.tri"))
if len(sys.argv) > 4:
    _lib.lib.mwt_set_tuning(int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]) if len(sys.argv) > 5 else 0)


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for mode in (0, 1):
    rays = mesh.raygen_device(mode, box, 0, 0, n)
    pts = rays[:, :2].contiguous()
    tid, _ = mesh.locate_device(pts)
    hist = new_histogram()
    print(f"mode {mode}:")
    print(f"  raygen (write rays)   {timeit(lambda: mesh.raygen_device(mode, box, 0, 0, n)):.3f} ms")
    print(f"  locate (k_locate)     {timeit(lambda: mesh.locate_device(pts)):.3f} ms")
    print(f"  walk, start given     {timeit(lambda: mesh.trace_device(rays, tid, want=('seg', 't', 'steps'))):.3f} ms")
    print(f"  locate+walk (loaded)  {timeit(lambda: mesh.trace_device(rays, None, want=('seg', 't', 'steps'))):.3f} ms")
    print(f"  fused generated       {timeit(lambda: mesh.trace_generated_device(mode, box, 0, 0, n, True, hist)):.3f} ms")
    print(f"  fused, no outputs     {timeit(lambda: mesh.trace_generated_device(mode, box, 0, 0, n, False, hist)):.3f} ms")
