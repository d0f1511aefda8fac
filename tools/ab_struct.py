"""A/B timing of the kd-tree / BVH kernels (the library is MWT_LIB_PATH's).

usage: python tools/ab_struct.py cfg kd_ct bvh_ct [n]
prints one JSON line: ms and rays/s per (structure, order), plus a digest of
every output array so builds can be checked for identical results.
"""
import hashlib
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2112_05570_b200 import _lib  # noqa: E402
from paper_2112_05570_b200.engine import DeviceBvh, DeviceKd, DeviceMesh  # noqa: E402
from paper_2112_05570_b200.formats import load_structure  # noqa: E402

cfg, kd_ct, bvh_ct = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 22
box = bench.CONFIGS[cfg][0]
d = os.path.join(ROOT, "fixtures", "data", cfg)
mesh = DeviceMesh.from_files(*bench.fixture(cfg, "mwt"))
structs = {"kd": DeviceKd(mesh, load_structure(os.path.join(d, f"kd_ct{kd_ct}.npz"))),
           "bvh": DeviceBvh(mesh, load_structure(os.path.join(d, f"bvh_ct{bvh_ct}.npz")))}
out = {"lib": os.path.relpath(_lib.LIB_PATH, ROOT), "cfg": cfg, "n": n}
for order in ("coherent", "iid"):
    rays = mesh.raygen_device(bench.mode_word(0, order), box, bench.SEED, 0, n)
    for name, st in structs.items():
        ms = bench._time_ms(lambda: st.trace_device(rays))
        r = st.trace_device(rays)
        torch.cuda.synchronize()
        h = hashlib.sha256()
        for k in sorted(r):
            h.update(r[k].cpu().numpy().tobytes())
        ops = sum(float(v.double().sum()) for k, v in r.items() if k in ("nodes", "ropes", "prims",
                                                                        "node_tests", "prim_tests"))
        out[f"{name}/{order}"] = {"ms": round(ms, 4), "grays_s": round(n / ms / 1e6, 3),
                                  "ops_per_ray": round(ops / n, 3), "digest": h.hexdigest()[:16]}
print(json.dumps(out))
