"""Launch the kd-tree and BVH kernels on one config's box-entry rays (for ncu).

usage: python tools/prof_struct.py cfg order n [kd_ct bvh_ct]
  e.g. ncu --set full -k regex:"k_kd|k_bvh" -s 2 -c 2 python tools/prof_struct.py floorplan64 iid 4194304 2 2
Each kernel runs three times (the first two are warm-up for a -s 2 skip).
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2112_05570_b200.engine import DeviceBvh, DeviceKd, DeviceMesh  # noqa: E402
from paper_2112_05570_b200.formats import load_structure  # noqa: E402

cfg, order, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
kd_ct = sys.argv[4] if len(sys.argv) > 4 else "2"
bvh_ct = sys.argv[5] if len(sys.argv) > 5 else "2"
box = bench.CONFIGS[cfg][0]
d = os.path.join(ROOT, "fixtures", "data", cfg)
mesh = DeviceMesh.from_files(*bench.fixture(cfg, "mwt"))
kd = DeviceKd(mesh, load_structure(os.path.join(d, f"kd_ct{kd_ct}.npz")))
bvh = DeviceBvh(mesh, load_structure(os.path.join(d, f"bvh_ct{bvh_ct}.npz")))
rays = mesh.raygen_device(bench.mode_word(0, order), box, bench.SEED, 0, n)
for st in (kd, kd, kd, bvh, bvh, bvh):
    r = st.trace_device(rays)
torch.cuda.synchronize()
k = kd.trace_device(rays)
b = bvh.trace_device(rays)
print("kd ops/ray", float(sum(k[x].double().sum() for x in ("nodes", "ropes", "prims"))) / n,
      "bvh ops/ray", float(sum(b[x].double().sum() for x in ("node_tests", "prim_tests"))) / n)
